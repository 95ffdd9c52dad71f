#!/usr/bin/env python
"""Dose-evaluation benchmark: d = A.x over the native-encoding DDM on 1..N B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--accum exact|fp32]
    python bench.py --impl reference ...      # the reference's own CPU path (oracle/_ref)

One step = one dose evaluation over the whole matrix (every rank's row shard).  Workload (N=1):
BASELINE.json configs[1], C2 = 8M voxels x 40k spots, ~3.2e9 nnz, binary16 values, u16 indices,
generated on the device (the reference's serial host generator would take ~7 min); x =
ddm::seeded_vector(40000, 42).  The matrix (12.9 GB) is ~100x the 126 MB L2, so no flush is
needed between steps ("inputs larger than L2").  --config c4 is the optimisation loop of
SURVEY 8(d): step k doses x_k = seeded_vector(196608, 1000 + k) (8 x cycled).

value    = SpMV effective GB/s = sum over ranks of ddm::traffic(dims, layout_of) bytes / step
           time (max over ranks, CUDA events, device-resident x/d).
e2e      = same metric through the public API with pinned HOST x and d: H2D x + kernels +
           D2H d inside the timed region.
roofline = the dominant kernel's algorithmic bytes / its CUDA-event duration vs the measured
           HBM copy peak (MEASURED_PEAKS.json).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c4", "c5"])
    ap.add_argument("--accum", default="exact", choices=["exact", "fp32"])
    ap.add_argument("--rows", type=int, default=0, help="override rows (testing)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-alt-fp32", action="store_true", help="skip the fp32-family side line")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--cpu-sample-rows", type=int, default=250_000)
    ap.add_argument("--e2e-steps", type=int, default=0, help="default: --steps")
    ap.add_argument("--engine", default="shard", choices=["shard", "multi"],
                    help="shard: one process per GPU (torchrun for N > 1); multi: one process "
                         "driving --gpus devices through the dg_multi handle (DG_BENCH_DEVICES="
                         "0,0,... lists them explicitly, e.g. virtual shards on one GPU)")
    ap.add_argument("--gather", default="peer", choices=["none", "peer", "nccl"],
                    help="--engine multi: the d gather of each step")
    return ap.parse_args()


def workload(cfg: str, rows_override: int = 0):
    from paper_2103_09683_b200 import profiles as P
    if cfg == "c1":
        ps = [P.c1()]
    elif cfg == "c2":
        ps = [P.c2()]
    elif cfg == "c4":
        ps = P.c4_beams()
    else:  # c5: the nine robust scenarios (separate matrices, evaluated back to back)
        ps = P.c5_scenarios()
    if rows_override:
        for p in ps:
            p.rows = rows_override
    return ps


def workload_desc(cfg, ps):
    return {"c1": "C1 synthetic DDM 1M voxels x 4,096 spots ~1% (configs[0])",
            "c2": "C2 clinical-scale synthetic DDM 8M voxels x 40k spots ~3.2e9 nnz, skewed "
                  "(configs[1])",
            "c4": "C4 6-beam hstack 2.97M voxels x 196,608 spots, U32 indices (configs[3])",
            "c5": "C5 robust planning: 9 scenarios x 88M voxels x 40k spots, each GPU holds 1/8 "
                  "of every scenario (configs[4])"}[cfg]


def measured_hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons, sampled every 100 ms.  Started before the warm-up
    (nvidia-smi's own start-up -- NVML init -- must not overlap the timed region); only the samples
    taken inside [mark_start, mark_stop] are reported (all of them if the region was shorter than
    one sampling period, with "in_region": false)."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.rows = []
        self.proc = None
        self.t0 = self.t1 = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(device)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append((time.time(), parts))

    def wait_ready(self, timeout: float = 5.0):
        """Block until nvidia-smi has produced its first sample (its start-up is over)."""
        end = time.time() + timeout
        while self.proc and not self.rows and time.time() < end:
            time.sleep(0.02)

    def mark_start(self):
        self.t0 = time.time()

    def mark_stop(self):
        self.t1 = time.time()

    def stop(self):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        rows = [r for t, r in self.rows
                if self.t0 is not None and self.t1 is not None and self.t0 <= t <= self.t1 + 0.1]
        in_region = bool(rows)
        if not rows:
            rows = [r for _, r in self.rows]
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows), "in_region": in_region}


# ---------------------------------------------------------------------- CPU baselines ------
def host_description() -> dict:
    """The box's host side: CPU model, sockets, NUMA nodes, threads, glibc."""
    import glob
    import platform
    d = {"threads": os.cpu_count()}
    try:
        with open("/proc/cpuinfo") as f:
            txt = f.read()
        models = [ln.split(":", 1)[1].strip() for ln in txt.splitlines() if ln.startswith("model name")]
        d["cpu_model"] = models[0] if models else platform.processor()
        phys = {ln.split(":", 1)[1].strip() for ln in txt.splitlines() if ln.startswith("physical id")}
        d["sockets"] = len(phys) or 1
    except Exception:
        d["cpu_model"] = platform.processor()
    d["numa_nodes"] = len(glob.glob("/sys/devices/system/node/node[0-9]*")) or 1
    try:
        d["glibc"] = os.confstr("CS_GNU_LIBC_VERSION")
    except Exception:
        d["glibc"] = " ".join(platform.libc_ver())
    return d


def cpu_oracle_single_thread(m, target_s: float = 3.0) -> dict:
    """ddm::run_bench(Algorithm::Oracle, workers 1) on the same sample -- SURVEY 8(d) CPU row (2)."""
    from oracle.oracle import Oracle, have_reference, traffic_bytes
    if not have_reference():
        return {"value": None, "error": "oracle/_ref not built"}
    orc = Oracle("reference")
    t1 = orc.run_bench(m, algorithm=0, lane_width=1, workers=1, reps=1, warmup=0,
                       vector_seed=42)["mean_seconds"]
    reps = max(1, min(20, int(target_s / max(t1, 1e-6))))
    r = orc.run_bench(m, algorithm=0, lane_width=1, workers=1, reps=reps, warmup=1,
                      vector_seed=42)
    b = traffic_bytes(m.rows, m.cols, m.nnz, 2, 2 if m.cols < 65536 else 4)
    return {"value": b / r["mean_seconds"] / 1e9, "unit": "GB/s", "cores": 1,
            "ms_per_eval": r["mean_seconds"] * 1e3,
            "sample": f"same sample, ddm::run_bench oracle workers=1 reps={reps} warmup=1"}


def cpu_reference_run(ps, sample_rows: int, reps: int, warmup: int,
                      target_s: float = 0.0, with_oracle_row: bool = False) -> dict:
    """The reference's own CPU dose path, unmodified (oracle/_ref = /root/reference/proj built
    by oracle/Makefile): ddm::generate on a row sample of the workload's profile, then
    ddm::run_bench(RowChunk, lane_width 32, workers = all host threads) -- bench.cpp:38-103.
    target_s > 0: reps chosen so the timed CPU work is about target_s seconds."""
    from oracle.oracle import Oracle, Profile, have_reference, traffic_bytes
    if len(ps) > 1 and len({p.cols for p in ps}) == 1 and ps[0].seed > 100:
        ps = ps[:1]  # C5: the scenarios are separate matrices; sample one of them
    cores = os.cpu_count() or 1
    kind = "reference" if have_reference() else "port"
    orc = Oracle(kind)
    sub = [Profile(sample_rows, p.cols, p.target_nnz_ratio, p.empty_row_fraction,
                   p.row_length_log_mean, p.row_length_log_sigma, p.locality_window, p.seed)
           for p in ps]
    parts = [orc.generate(p) for p in sub]
    m = parts[0] if len(parts) == 1 else hstack(parts)
    if kind == "reference":
        if target_s > 0:  # calibrate on one evaluation
            t1 = orc.run_bench(m, algorithm=1, lane_width=32, workers=cores, reps=1, warmup=1,
                               vector_seed=42)["mean_seconds"]
            reps = max(3, min(400, int(target_s / max(t1, 1e-6)) + 1))
        r = orc.run_bench(m, algorithm=1, lane_width=32, workers=cores, reps=reps,
                          warmup=warmup, vector_seed=42)
        mean_s = r["mean_seconds"]
    else:
        import numpy as np
        x = orc.seeded_vector(m.cols, 42)
        for _ in range(warmup):
            orc.spmv_rowchunk(m, x, 32, cores)
        t0 = time.perf_counter()
        for _ in range(reps):
            orc.spmv_rowchunk(m, x, 32, cores)
        mean_s = (time.perf_counter() - t0) / reps
        del np
    vb, ib = 2, (2 if m.cols < 65536 else 4)
    b = traffic_bytes(m.rows, m.cols, m.nnz, vb, ib)
    extra = {}
    if with_oracle_row:
        try:
            extra["oracle_workers1"] = cpu_oracle_single_thread(m)
        except Exception as ex:  # reported, never silently replaced
            extra["oracle_workers1"] = {"value": None, "error": str(ex)[:200]}
    return {"value": b / mean_s / 1e9, "unit": "GB/s", "cores": cores, "kind": kind,
            "ms_per_eval": mean_s * 1e3, "model_bytes": b, "host": host_description(), **extra,
            "sample": f"ddm::generate rows={sample_rows} of the workload profile "
                      f"({m.nnz} nnz, {b / 1e9:.3f} GB model bytes), ddm::run_bench rowchunk "
                      f"L=32 workers={cores}, reps={reps} warmup={warmup}"}


def hstack(parts):
    """Column-wise hstack of per-beam CSR matrices (C4's multi-beam plan)."""
    import numpy as np
    from oracle.oracle import U32, Csr
    rows = parts[0].rows
    off, lens = 0, []
    for p in parts:
        lens.append(np.diff(p.row_ptr.astype(np.int64)))
    tot = np.sum(lens, axis=0)
    rp = np.zeros(rows + 1, dtype=np.uint64)
    np.cumsum(tot, out=rp[1:])
    col = np.empty(int(rp[-1]), dtype=np.uint32)
    val = np.empty(int(rp[-1]), dtype=parts[0].values.dtype)
    pos = rp[:-1].astype(np.int64).copy()
    for p, ln in zip(parts, lens):
        for r in np.nonzero(ln)[0]:
            s, e = int(p.row_ptr[r]), int(p.row_ptr[r + 1])
            col[pos[r]:pos[r] + e - s] = p.col[s:e] + off
            val[pos[r]:pos[r] + e - s] = p.values[s:e]
            pos[r] += e - s
        off += p.cols
    return Csr(rows, off, parts[0].precision, U32, rp, col, val)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    ps = workload(args.config, args.rows)
    r = cpu_reference_run(ps, args.cpu_sample_rows, max(args.steps, 1), max(args.warmup, 0))
    line = {"impl": "reference", "metric": metric_name(args.config), "value": r["value"],
            "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": r["ms_per_eval"], "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference generator)",
            "config": {"workload": workload_desc(args.config, ps), "sample_rows": args.cpu_sample_rows},
            "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample", "host")},
            "e2e": {"value": r["value"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def metric_name(cfg):
    return "SpMV effective GB/s per dose eval (ms per dose eval in ms_per_step)"


# ---------------------------------------------------------------------- our arm ------------
def build_engines(args, dg, rank, world, local, accum):
    """This rank's resident matrices.  C1/C2/C4: one matrix, row-sharded nnz-balanced over the
    ranks (strong scaling).  C5: the nine robust scenarios, each cut into 8 nnz-balanced row
    shards; rank r holds shard r of every scenario -- one GPU's share of the 8-GPU residency
    (weak scaling: per-GPU work is fixed)."""
    ps = workload(args.config, args.rows)
    cols = ps[0].cols if args.config == "c5" else sum(p.cols for p in ps)  # C5: not hstacked
    bpn = 2 + (2 if cols < 65536 else 4)
    engines = []
    if args.config == "c5":
        if world > 8:
            raise SystemExit("c5 is laid out over 8 GPUs")
        for p in ps:
            lens = dg.generated_row_lengths(p, 0, p.rows, device=local)
            b = dg.partition_lengths(lens, 8, bpn)
            engines.append(dg.DoseEngine.generate(p, row_begin=int(b[rank]), row_end=int(b[rank + 1]),
                                                  device=local, accumulation=accum))
        return ps, cols, engines, None
    rows = ps[0].rows
    bounds = None
    if world > 1:
        lens = dg.generated_row_lengths(ps, 0, rows, device=local)
        bounds = dg.partition_lengths(lens, world, bpn)
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    else:
        r0, r1 = 0, rows
    engines.append(dg.DoseEngine.generate(ps, row_begin=r0, row_end=r1, device=local,
                                          accumulation=accum))
    return ps, cols, engines, bounds


def run_ours(args):
    import numpy as np
    import torch

    import paper_2103_09683_b200 as dg

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # DG_BENCH_ONE_DEVICE=1 (+ --dist-backend gloo): every rank on cuda:0 -- exercises the N > 1
    # orchestration on a single-GPU box; the timing is then not a scaling measurement
    if os.environ.get("DG_BENCH_ONE_DEVICE") == "1":
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(args.dist_backend)

    accum = dg.ACCUM_EXACT if args.accum == "exact" else dg.ACCUM_FP32
    t0 = time.time()
    ps, cols, engines, bounds = build_engines(args, dg, rank, world, local, accum)
    setup_s = time.time() - t0
    rows_total = ps[0].rows * (len(ps) if args.config == "c5" else 1)
    # C4 is an optimisation loop: evaluation k doses x_k = seeded_vector(cols, 1000 + k);
    # the steps cycle through 8 such x (device-resident for `value`, uploaded per step for e2e).
    # Every other config doses seeded_vector(cols, 42).
    x_seeds = [1000 + k for k in range(8)] if args.config == "c4" else [42]
    x_hosts = [dg.seeded_vector(cols, sd) for sd in x_seeds]
    x_host = x_hosts[0]
    xs = [torch.from_numpy(xv).cuda() for xv in x_hosts]
    x = xs[0]
    x_ctr = [0]

    def next_x():
        k = x_ctr[0] % len(xs)
        x_ctr[0] += 1
        return k
    ys = [torch.empty(e.info["rows"], dtype=torch.float64, device="cuda") for e in engines]
    # a real (non-legacy) stream shared by our kernels and the timing events
    torch_stream = torch.cuda.Stream()
    torch.cuda.set_stream(torch_stream)
    stream = torch_stream.cuda_stream

    def step(profile=False, engs=None):
        xk = xs[next_x()]
        for e, y in zip(engs or engines, ys):
            e.dose_device(xk.data_ptr(), cols, y.data_ptr(), stream=stream, sync=False,
                          profile=profile)

    def timed(fn, n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b)

    clocks = ClockSampler(local)
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    clocks.wait_ready()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.mark_start()
    ms = timed(step, args.steps)
    clocks.mark_stop()
    clk = clocks.stop()
    if dist:
        dist.barrier()

    # dominant kernel: CUDA events per launch (same stream), right after the timed region
    prof_steps = min(args.steps, 10)
    per = {}
    for _ in range(prof_steps):
        for e, y in zip(engines, ys):
            e.dose_device(x.data_ptr(), cols, y.data_ptr(), stream=stream, sync=False, profile=True)
            for k in e.kernel_times():
                d = per.setdefault(k["name"], {"ms": 0.0, "bytes": 0})
                d["ms"] += k["ms"] / prof_steps
                d["bytes"] += k["bytes"] / prof_steps
    dom_name, dom = max(per.items(), key=lambda kv: kv[1]["ms"])

    # end to end through the public API: pinned host x and d, H2D + kernels + D2H timed
    e2e_steps = args.e2e_steps or args.steps
    xhs = [torch.from_numpy(xv).pin_memory() for xv in x_hosts]
    yhs = [torch.empty(e.info["rows"], dtype=torch.float64).pin_memory() for e in engines]
    e2e_last = [0]

    def e2e_step(engs=None):
        k = next_x()
        e2e_last[0] = k
        for e, yh in zip(engs or engines, yhs):
            e.dose_host_ptrs(xhs[k].data_ptr(), cols, yh.data_ptr(), stream=stream)

    e2e_step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e2e_ms = timed(e2e_step, e2e_steps)
    for e, y in zip(engines, ys):  # the device path on the last e2e step's x, for the check below
        e.dose_device(xs[e2e_last[0]].data_ptr(), cols, y.data_ptr(), stream=stream, sync=True)
    torch.cuda.synchronize()
    for yh, y in zip(yhs, ys):
        assert np.array_equal(yh.numpy().view(np.uint64), y.cpu().numpy().view(np.uint64)), \
            "host-path d differs from device-path d"

    # N > 1 (C2/C3): the d slices all-gathered over NCCL into the full d on every rank (8(e)),
    # timed separately from the sharded-resident step
    gather_ms = fused_ms = blocks_ms = 0.0
    if dist and bounds is not None:
        from paper_2103_09683_b200.sharded import gather_dose
        for _ in range(2):
            step()
            gather_dose(ys[0], bounds)
        torch.cuda.synchronize()
        dist.barrier()
        full = [None]

        def step_gather():
            step()
            full[0] = gather_dose(ys[0], bounds)

        gather_ms = timed(step_gather, e2e_steps)
        assert full[0].numel() == ps[0].rows

        # the same exchange fused into the dose kernels: rows stored into every rank's full d over
        # peer memory (CUDA IPC mappings), then a one-element all_reduce as the device-side
        # barrier that orders every rank's stores before the step ends
        # mode "blocks": the same buffers filled by copy-engine DMA of each row block as the tile
        # kernel finishes it (dg_set_block_targets)
        from paper_2103_09683_b200.sharded import FusedGather
        if FusedGather.preflight(local):  # same answer on every rank
            for mode in ("epilogue", "blocks"):
                fg = FusedGather(engines[0], bounds, local, mode=mode)
                flag = torch.zeros(1, dtype=torch.float64, device="cuda")

                def step_fused():
                    step()
                    dist.all_reduce(flag)

                for _ in range(2):
                    step_fused()
                torch.cuda.synchronize()
                dist.barrier()
                t_mode = timed(step_fused, e2e_steps)
                dist.barrier()
                assert torch.equal(fg.full.view(torch.int64), full[0].view(torch.int64)), \
                    f"fused gather ({mode}) differs from the NCCL all-gather"
                fg.close()
                if mode == "epilogue":
                    fused_ms = t_mode
                else:
                    blocks_ms = t_mode
        else:
            fused_ms = blocks_ms = -1.0  # CUDA IPC unavailable between these processes

    model_bytes = sum(e.info["model_bytes"] for e in engines)
    nnz = sum(e.info["nnz"] for e in engines)
    lrows = sum(e.info["rows"] for e in engines)
    vals = torch.tensor([ms, e2e_ms, gather_ms, fused_ms, blocks_ms], dtype=torch.float64,
                        device="cuda")
    sums = torch.tensor([float(model_bytes), float(nnz), 8.0 * cols * len(engines), 8.0 * lrows],
                        dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
        dist.all_reduce(sums, op=dist.ReduceOp.SUM)
    ms, e2e_ms, gather_ms, fused_ms, blocks_ms = vals.tolist()
    total_bytes, total_nnz, h2d, d2h = sums.tolist()
    ms_step = ms / args.steps
    e2e_step_ms = e2e_ms / e2e_steps

    if rank != 0:
        for e in engines:
            e.close()
        if dist:
            dist.destroy_process_group()
        return
    peak, peak_kind = measured_hbm_peak()
    achieved = dom["bytes"] / (dom["ms"] * 1e-3) / 1e9
    traffic = traffic_step = None
    tf = os.path.join(ROOT, "profiles", "dram_bytes_per_launch.json")
    if os.path.exists(tf) and world == 1 and not args.rows:  # profiled: the full 1-GPU workload
        try:
            tj = json.load(open(tf))

            def tget(name):
                return tj.get(f"{args.config}:{args.accum}:{name}",
                              tj.get(f"{args.config}:{args.accum}:{name.split('[')[0]}"))
            traffic = tget(dom_name)
            # DRAM bytes of the whole dose (every kernel with an ncu figure): with the value
            # stream (implied column words) it is below the reference-model bytes
            tk = [tget(k) for k in per]
            traffic_step = int(sum(tk)) if tk and all(v is not None for v in tk) else None
        except Exception:
            traffic = None
    info = engines[0].info
    line = {
        "metric": metric_name(args.config),
        "value": total_bytes / (ms_step * 1e-3) / 1e9,
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": max(args.warmup, 3),
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "weak" if args.config == "c5" else "strong",
        "vs_baseline": None,
        "dtype": "f64" if accum == dg.ACCUM_EXACT else "f32",
        "data": "synthetic (row-parallel device generator, reference profile statistics)",
        "config": {"workload": workload_desc(args.config, ps), "rows": rows_total, "cols": cols,
                   "nnz": int(total_nnz), "value_precision": "binary16",
                   "index_bytes": info["index_bytes"],
                   "accumulation": "exact fp64, bit-identical to ddm::spmv_rowchunk L=32"
                   if accum == dg.ACCUM_EXACT else "fp32 (tol 1e-5 * max|d|)",
                   "parallelism": (f"9 scenarios x 1/8 row shard per GPU x{world}"
                                   if args.config == "c5" else
                                   f"row-shard x{world} (nnz-balanced)"),
                   "model_bytes_per_step": int(total_bytes), "l2": "inputs larger than L2",
                   "x": ("x_k = seeded_vector(cols, 1000 + k), k = step mod 8 (optimisation loop)"
                         if args.config == "c4" else "seeded_vector(cols, 42)"),
                   "setup_s": round(setup_s, 2)},
        "frac_of_8TBps": total_bytes / (ms_step * 1e-3) / 8e12 / world,
        "frac_of_measured_hbm": total_bytes / (ms_step * 1e-3) / 1e9 / peak / world,
        "roofline": {"bound": "hbm", "kernel": dom_name, "achieved": achieved, "peak": peak,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "traffic_step_ncu": traffic_step,
                     "note": "achieved / value count the reference model's bytes ((vb+ib)*nnz + "
                             "16*rows + 8*cols, perf_model.cpp:41-54); contiguous rows are "
                             "streamed without their implied column words and U32 columns as "
                             "16-bit window slots, so the DRAM bytes (traffic*) are fewer",
                     "bytes_per_launch": dom["bytes"] / len(engines),
                     "ms_per_launch": dom["ms"] / len(engines),
                     "share_of_step": dom["ms"] / (ms / args.steps if world == 1 else ms_step),
                     "kernels": {k: {"ms": round(v["ms"], 4), "bytes": int(v["bytes"])}
                                 for k, v in per.items()}},
        "e2e": {"value": total_bytes / (e2e_step_ms * 1e-3) / 1e9, "unit": "GB/s",
                "ms_per_step": e2e_step_ms, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": sum(int(e.info["n_kernels"]) for e in engines) * args.steps * world,
        "ms_per_step_gathered": (gather_ms / e2e_steps) if gather_ms else None,
        "ms_per_step_gathered_fused": (fused_ms / e2e_steps) if fused_ms > 0 else
                                      ("unavailable: CUDA IPC" if fused_ms < 0 else None),
        "ms_per_step_gathered_blocks": (blocks_ms / e2e_steps) if blocks_ms > 0 else
                                       ("unavailable: CUDA IPC" if blocks_ms < 0 else None),
        "clocks": clk,
    }
    if args.config == "c5":
        line["ms_per_scenario"] = ms_step / len(engines)
    if world == 1 and accum == dg.ACCUM_EXACT and not args.no_alt_fp32 and args.config != "c5":
        # the north_star tolerance family on the same workload, reported beside the exact one
        for e in engines:
            e.close()
        _, _, fengs, _ = build_engines(args, dg, rank, world, local, dg.ACCUM_FP32)
        for _ in range(3):
            step(engs=fengs)
        torch.cuda.synchronize()
        fms = timed(lambda: step(engs=fengs), args.steps) / args.steps
        e2e_step(fengs)
        fe2e = timed(lambda: e2e_step(fengs), e2e_steps) / e2e_steps
        line["alt_fp32"] = {"dtype": "f32", "tolerance": "per-voxel |d - d_ref| <= 1e-5 max|d_ref|",
                            "value": total_bytes / (fms * 1e-3) / 1e9, "ms_per_step": fms,
                            "frac_of_measured_hbm": total_bytes / (fms * 1e-3) / 1e9 / peak,
                            "e2e": {"value": total_bytes / (fe2e * 1e-3) / 1e9, "ms_per_step": fe2e}}
        engines = fengs
    if world == 1 and not args.no_cpu_baseline:
        try:
            r = cpu_reference_run(ps, args.cpu_sample_rows, 5, 1, target_s=10.0,
                                  with_oracle_row=True)
            line["cpu_baseline"] = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample",
                                                      "host", "oracle_workers1") if k in r}
        except Exception as ex:  # reported, never silently replaced
            line["cpu_baseline"] = {"value": None, "error": str(ex)[:200]}
    else:
        line["cpu_baseline"] = None
    print(json.dumps(line), flush=True)
    for e in engines:
        e.close()
    if dist:
        dist.destroy_process_group()


def run_multi(args):
    """--engine multi: one process drives every device through the dg_multi handle (the C-ABI
    multi-GPU product path).  A step = dg_multi_dose with x on devices[0]: x peer-copied to every
    device, the shards' doses run concurrently, then the --gather exchange; timed per step with
    CUDA events on every device (max over devices, dg_multi_last_timing)."""
    import numpy as np
    import torch

    import paper_2103_09683_b200 as dg

    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        raise SystemExit("--engine multi is one process (no torchrun)")
    devs = os.environ.get("DG_BENCH_DEVICES")
    devices = [int(d) for d in devs.split(",")] if devs else list(range(args.gpus))
    gather = {"none": dg.GATHER_NONE, "peer": dg.GATHER_PEER, "nccl": dg.GATHER_NCCL}[args.gather]
    accum = dg.ACCUM_EXACT if args.accum == "exact" else dg.ACCUM_FP32
    ps = workload(args.config, args.rows)
    if args.config == "c5":
        raise SystemExit("--engine multi: c1 / c2 / c4")
    cols = sum(p.cols for p in ps)
    torch.cuda.set_device(devices[0])
    t0 = time.time()
    m = dg.MultiDoseEngine.generate(ps, devices, gather=gather, accumulation=accum)
    setup_s = time.time() - t0
    shards = [m.shard(i) for i in range(m.n_shards)]
    model_bytes = sum(e.info["model_bytes"] for e in shards)
    x_host = dg.seeded_vector(cols, 42)
    x = torch.from_numpy(x_host).cuda()

    def run(n, fn):
        tot = ker = 0.0
        for _ in range(n):
            fn()
            t = m.last_timing()
            tot += t["ms_total"]
            ker += t["ms_kernels"]
        return tot, ker

    for _ in range(max(args.warmup, 3)):
        m.dose_device(x.data_ptr(), cols)
    clocks = ClockSampler(devices[0])
    clocks.wait_ready()
    clocks.mark_start()
    ms, kms = run(args.steps, lambda: m.dose_device(x.data_ptr(), cols))
    clocks.mark_stop()
    clk = clocks.stop()
    xh = torch.from_numpy(x_host).pin_memory()
    yh = torch.empty(m.rows, dtype=torch.float64).pin_memory()
    m.dose_host_ptrs(xh.data_ptr(), cols, yh.data_ptr())
    e2e_ms, _ = run(args.steps, lambda: m.dose_host_ptrs(xh.data_ptr(), cols, yh.data_ptr()))
    full, _ = m.device_d(0)
    if gather != dg.GATHER_NONE:
        d0 = torch.empty(m.rows, dtype=torch.float64, device=f"cuda:{devices[0]}")
        torch.cuda.synchronize()
        d0.copy_(torch.as_tensor(_DevView(full, m.rows), device=f"cuda:{devices[0]}"))
        assert np.array_equal(d0.cpu().numpy().view(np.uint64), yh.numpy().view(np.uint64)), \
            "gathered d on device 0 differs from the host d"
    ms_step, e2e_step_ms = ms / args.steps, e2e_ms / args.steps
    n_phys = len(set(devices))
    line = {
        "metric": metric_name(args.config), "engine": "multi (dg_multi, one process)",
        "value": model_bytes / (ms_step * 1e-3) / 1e9, "unit": "GB/s", "n_gpus": n_phys,
        "shards": len(devices), "devices": devices, "gather": args.gather,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms_step,
        "ms_per_step_kernels": kms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64" if accum == dg.ACCUM_EXACT else "f32",
        "data": "synthetic (row-parallel device generator, reference profile statistics)",
        "config": {"workload": workload_desc(args.config, ps), "rows": m.rows, "cols": cols,
                   "parallelism": f"row-shard x{len(devices)} over {n_phys} device(s), "
                                  f"gather {args.gather}",
                   "model_bytes_per_step": int(model_bytes), "l2": "inputs larger than L2",
                   "setup_s": round(setup_s, 2)},
        "e2e": {"value": model_bytes / (e2e_step_ms * 1e-3) / 1e9, "unit": "GB/s",
                "ms_per_step": e2e_step_ms, "h2d_bytes_per_step": 8 * cols * len(devices),
                "d2h_bytes_per_step": 8 * m.rows},
        "gpu_launches": sum(int(e.info["n_kernels"]) for e in shards) * args.steps,
        "clocks": clk, "cpu_baseline": None,
    }
    print(json.dumps(line), flush=True)
    m.close()


class _DevView:
    """A raw device pointer as a __cuda_array_interface__ (float64[n])."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False),
                                         "version": 2, "strides": None}


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    elif args.engine == "multi":
        run_multi(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
