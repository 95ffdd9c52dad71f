#!/usr/bin/env python
"""Tile-timeline diagnostic (DG_TRACE): where does the tile kernel lose time on a workload?

    DG_TRACE=1 python scripts/trace_tiles.py [--config c2] [--accum exact]

Prints the CTA end-time spread (tail), the fraction of warp time spent waiting for a window
buffer, and tile durations by kind (global-x vs windowed)."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("DG_TRACE", "1")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--accum", default="exact")
    ap.add_argument("--rows", type=int, default=0)
    a = ap.parse_args()
    import torch

    import bench
    import paper_2103_09683_b200 as dg
    ps = bench.workload(a.config, a.rows)
    acc = dg.ACCUM_EXACT if a.accum == "exact" else dg.ACCUM_FP32
    e = dg.DoseEngine.generate(ps, device=0, accumulation=acc)
    cols = sum(p.cols for p in ps)
    x = torch.from_numpy(dg.seeded_vector(cols, 42)).cuda()
    y = torch.empty(e.info["rows"], dtype=torch.float64, device="cuda")
    for _ in range(3):
        e.dose_device(x.data_ptr(), cols, y.data_ptr(), sync=True)
    st = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st[0].record()
    e.dose_device(x.data_ptr(), cols, y.data_ptr(), sync=True)
    st[1].record()
    torch.cuda.synchronize()
    tr = e.debug_trace().astype(np.int64)
    sms = 148
    cta = tr[:4 * sms].reshape(sms, 4)
    tl = tr[4 * sms:].reshape(-1, 3)
    t0 = cta[:, 0].min()
    start = (cta[:, 0] - t0) / 1e3
    end = (cta[:, 1] - t0) / 1e3
    print(f"dose {st[0].elapsed_time(st[1]):.3f} ms (events, incl. memsets); tiles {len(tl)}")
    print(f"CTA start spread {start.max():.1f} us; end: min {end.min():.1f} median "
          f"{np.median(end):.1f} max {end.max():.1f} us")
    print(f"tail (max end - median end) {end.max() - np.median(end):.1f} us, "
          f"(max - min) {end.max() - end.min():.1f} us")
    wait = cta[:, 2].sum() / max(1, cta[:, 3].sum())
    print(f"warp time waiting for a window buffer: {100 * wait:.1f}%  (per CTA max "
          f"{100 * (cta[:, 2] / np.maximum(1, cta[:, 3])).max():.1f}%)")
    claim = (tl[:, 0] - t0) / 1e3
    fin = (tl[:, 1] - t0) / 1e3
    dur = fin - claim
    meta = tl[:, 2]
    glob = (meta >> 62) & 1
    nseg = (meta >> 16) & 0xFFFFFF
    for k, name in ((1, "global-x"), (0, "windowed")):
        m = glob == k
        if m.any():
            print(f"{name:9s} tiles {m.sum():5d}: dur us median {np.median(dur[m]):.1f} "
                  f"p90 {np.percentile(dur[m], 90):.1f} max {dur[m].max():.1f}; segs median "
                  f"{np.median(nseg[m]):.0f}")
    last = np.argsort(fin)[-12:]
    print("last tiles to finish (idx, kind, claim us, finish us, segs):")
    for i in last:
        print(f"  {i:5d} {'G' if glob[i] else 'W'} {claim[i]:8.1f} {fin[i]:8.1f} {nseg[i]:5d}")
    # concurrency profile: tiles in progress over time (10 us bins)
    T = end.max()
    bins = np.arange(0, T + 10, 10)
    act = [(np.sum((claim <= b) & (fin > b))) for b in bins]
    print("tiles in flight every 10 us:", " ".join(str(v) for v in act))
    e.close()


if __name__ == "__main__":
    main()
