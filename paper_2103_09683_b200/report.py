"""GPU rows in the reference's BenchReport format.

Mirrors ``ddm::BenchReport`` / ``ddm::run_bench`` / ``ddm::render_csv``
(include/ddm/bench.hpp:36-74, src/bench.cpp:38-103,141-153) so the reference's own report tooling
can audit GPU parity and throughput side by side with its CPU engines: same columns, same
checksum-drift abort (bench.cpp:72-78), same perf-model figures (traffic(dims_of, layout_of), OI),
and the same identity gflops == oi * gbps held bit for bit.  The algorithm column reads "cuda".
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass
from typing import Iterable, Optional

import numpy as np

from .dose import ACCUM_EXACT, DoseEngine, Errc, Error, checksum_bits, seeded_vector

_PREC = {2: "half", 4: "single", 8: "double"}


@dataclass
class BenchReport:
    """ddm::BenchReport (bench.hpp:36-50)."""
    matrix_label: str
    algorithm: str
    precision: str
    lane_width: int
    chunk_count: int
    workers: int
    repetitions: int
    mean_seconds: float
    min_seconds: float
    gflops: float
    effective_gbps: float
    operational_intensity: float
    output_checksum: int


def run_bench_gpu(engine: DoseEngine, label: str, *, repetitions: int = 100, warmup: int = 3,
                  vector_seed: int = 42, x: Optional[np.ndarray] = None) -> BenchReport:
    """ddm::run_bench (bench.cpp:38-103) for the GPU engine: x = seeded_vector(cols, seed), warm-up
    runs, then timed runs through the host-facing dose (the reference returns d on the host, so
    the timed region includes the upload of x and the download of d)."""
    if repetitions == 0:
        raise Error(1 + Errc.InvalidConfig, "repetitions must be at least 1")
    info = engine.info
    if x is None:
        x = seeded_vector(info["cols"], vector_seed)
    y = np.empty(info["rows"], dtype=np.float64)
    for _ in range(warmup):
        engine.dose(x, out=y)
    total = 0.0
    best = 0.0
    checksum = 0
    for rep in range(repetitions):
        t0 = time.perf_counter()
        engine.dose(x, out=y)
        el = time.perf_counter() - t0
        total += el
        best = el if rep == 0 else min(best, el)
        s = checksum_bits(y)
        if rep == 0:
            checksum = s
        elif s != checksum:  # bench.cpp:72-78
            raise Error(1 + Errc.ValidationFailure,
                        f"output checksum changed between repetitions ({checksum:016x} vs {s:016x})")
    mean = total / repetitions
    if not mean > 0.0:
        raise Error(1 + Errc.ZeroDuration, "timed region below clock resolution")
    vb, ib = info["value_bytes"], info["index_bytes"]
    total_bytes = (vb + ib) * info["nnz"] + 16 * info["rows"] + 8 * info["cols"]  # layout_of
    flops = 2 * info["nnz"]
    oi = flops / total_bytes  # operational_intensity (perf_model.cpp:56-60)
    gbps = total_bytes / mean * 1e-9
    return BenchReport(label, "cuda", _PREC[vb], info["lane_width"], 0, 1, repetitions, mean, best,
                       oi * gbps, gbps, oi, checksum)


def _fmt(v) -> str:
    """fmt's "{}" for the CSV cells: shortest round-trip decimal for doubles."""
    if isinstance(v, float):
        if math.isfinite(v) and v == int(v) and abs(v) < 1e16:
            return str(int(v))
        return repr(v)
    return str(v)


CSV_HEADER = ("matrix,algorithm,precision,lane_width,chunk_count,workers,repetitions,"
              "mean_seconds,min_seconds,gflops,effective_gbps,operational_intensity,"
              "output_checksum\n")


def render_csv(reports: Iterable[BenchReport]) -> str:
    """ddm::render_csv (bench.cpp:141-153)."""
    out = [CSV_HEADER]
    for r in reports:
        cells = [r.matrix_label, r.algorithm, r.precision, r.lane_width, r.chunk_count, r.workers,
                 r.repetitions, r.mean_seconds, r.min_seconds, r.gflops, r.effective_gbps,
                 r.operational_intensity]
        out.append(",".join(_fmt(c) for c in cells) + f",{r.output_checksum:016x}\n")
    return "".join(out)
