#!/usr/bin/env python
"""C3 on one GPU: the C2 matrix cut into G nnz-balanced row shards (exactly the shards
`bench.py --gpus G` gives each rank), each generated and timed in turn on cuda:0.

    python scripts/virtual_shards.py [--gpus 2 4 8] [--steps 50]

Per shard: kernel-only ms per dose (CUDA events, device-resident x and d).  The implied G-GPU
step is the max over shards (the bench's max-over-ranks rule) -- without the NVLink exchange,
which only the gathered variants need.  One JSON line per G."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2103_09683_b200 as dg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, nargs="+", default=[2, 4, 8])
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--config", default="c2")
    a = ap.parse_args()
    ps = bench.workload(a.config)
    rows, cols = ps[0].rows, sum(p.cols for p in ps)
    bpn = 2 + (2 if cols < 65536 else 4)
    lens = dg.generated_row_lengths(ps, 0, rows, device=0)
    x = torch.from_numpy(dg.seeded_vector(cols, 42)).cuda()
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    total = dg.traffic_bytes(rows, cols, int(lens.sum()), 2, bpn - 2)
    for G in a.gpus:
        b = dg.partition_lengths(lens, G, bpn)
        per = []
        for g in range(G):
            e = dg.DoseEngine.generate(ps, row_begin=int(b[g]), row_end=int(b[g + 1]), device=0)
            y = torch.empty(e.info["rows"], dtype=torch.float64, device="cuda")

            def step():
                e.dose_device(x.data_ptr(), cols, y.data_ptr(), stream=st.cuda_stream, sync=False)

            for _ in range(5):
                step()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            t0.record()
            for _ in range(a.steps):
                step()
            t1.record()
            torch.cuda.synchronize()
            ms = t0.elapsed_time(t1) / a.steps
            per.append({"shard": g, "rows": e.info["rows"], "nnz": e.info["nnz"],
                        "model_bytes": e.info["model_bytes"], "ms": round(ms, 4),
                        "gbps": round(e.info["model_bytes"] / ms / 1e6, 1)})
            e.close()
            del y
        worst = max(p["ms"] for p in per)
        shard_bytes = sum(p["model_bytes"] for p in per)
        print(json.dumps({"config": a.config, "gpus": G, "implied_ms_per_step": worst,
                          "implied_aggregate_gbps": round(shard_bytes / worst / 1e6, 1),
                          "single_matrix_model_bytes": total, "shards": per}), flush=True)


if __name__ == "__main__":
    main()
