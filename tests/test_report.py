"""GPU rows in the reference's BenchReport CSV: the CSV is byte-identical to
ddm::render_csv for the same field values (CPU), and a GPU report on the liver desk matrix carries
the reference engine's checksum and the gflops == oi * gbps identity (GPU)."""
import ctypes as C

import numpy as np
import pytest

import paper_2103_09683_b200 as dg
from paper_2103_09683_b200.report import BenchReport, render_csv, run_bench_gpu


def _ref_row(ref, r: BenchReport) -> str:
    f = ref.lib.ref_render_csv_row
    f.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                  C.c_double, C.c_double, C.c_double, C.c_double, C.c_double, C.c_uint64,
                  C.c_char_p, C.c_uint64]
    buf = C.create_string_buffer(4096)
    prec = {"half": 0, "single": 1, "double": 2}[r.precision]
    assert f(r.matrix_label.encode(), 1, prec, r.lane_width, r.chunk_count, r.workers,
             r.repetitions, r.mean_seconds, r.min_seconds, r.gflops, r.effective_gbps,
             r.operational_intensity, r.output_checksum, buf, 4096) == 0
    return buf.value.decode()


@pytest.mark.parametrize("vals", [
    (0.0123, 0.011, 1.25, 2.5, 0.5),
    (2.9e-3, 2.8e-3, 2210.4839248, 4455.31, 0.4950012),
    (1.0, 1e-05, 123456789.0, 1e+16, 3.0),
    (7.000000000000001e-06, 3e-21, 0.1, 0.30000000000000004, 0.33233),
])
def test_csv_is_byte_identical_to_reference(ref, vals):
    mean, mn, gflops, gbps, oi = vals
    r = BenchReport("liver-desk", "rowchunk", "half", 32, 0, 16, 100, mean, mn, gflops, gbps, oi,
                    0x0123456789ABCDEF)
    assert render_csv([r]) == _ref_row(ref, r)


@pytest.mark.gpu
def test_gpu_report_row(port, golden):
    from oracle.oracle import liver_desk
    m = port.generate(liver_desk())
    cm = dg.CsrMatrix(m.rows, m.cols, m.index_width, m.row_ptr, m.col, m.values, m.precision)
    with dg.DoseEngine.from_csr(cm) as e:
        r = run_bench_gpu(e, "liver-desk", repetitions=5, warmup=1)
    assert f"{r.output_checksum:016x}" == golden["liver-desk"]["rowchunk"]["32"]
    assert r.gflops == r.operational_intensity * r.effective_gbps  # bench.hpp:33-35 identity
    assert r.algorithm == "cuda" and r.lane_width == 32 and r.precision == "half"
    line = render_csv([r]).splitlines()[1].split(",")
    assert line[1] == "cuda" and line[-1] == golden["liver-desk"]["rowchunk"]["32"]
