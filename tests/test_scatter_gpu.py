"""The column-scatter comparator (the paper's "GPU Baseline" done atomic-free):
d bit-identical to ddm::spmv_scatter_baseline for the same chunk_count, on the reference's own
matrices; and the gather path (the product) faster than the scatter on a C2-shaped sample."""
import os

import numpy as np
import pytest

import paper_2103_09683_b200 as dg
from paper_2103_09683_b200.dose import ScatterEngine, spmv_scatter_baseline
from oracle.oracle import DOUBLE, SINGLE, U32, Csr, liver_desk, prostate_desk

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def to_dg(m: Csr) -> dg.CsrMatrix:
    return dg.CsrMatrix(m.rows, m.cols, m.index_width, m.row_ptr, m.col, m.values, m.precision)


@pytest.mark.parametrize("gen", [liver_desk, prostate_desk])
def test_scatter_matches_reference_every_chunk_count(ref, gen):
    m = ref.generate(gen())
    x = ref.seeded_vector(m.cols, 42)
    for chunks in (1, 2, 5, 64, 300):
        want = ref.spmv_scatter(m, x, chunks, 4)
        got = spmv_scatter_baseline(to_dg(m), x, chunks)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), chunks


@pytest.mark.parametrize("prec", [SINGLE, DOUBLE])
def test_scatter_other_precisions_and_integer_exactness(ref, prec):
    z = np.load(os.path.join(HERE, "golden", f"integer_{prec}.npz"))
    m = Csr(300, 120, prec, U32, z["row_ptr"], z["col"], z["values"])
    for chunks in (1, 6):
        got = spmv_scatter_baseline(to_dg(m), z["x"], chunks)
        assert np.array_equal(got.view(np.uint64), z["y"].view(np.uint64))
    m2 = ref.generate(liver_desk(), prec)
    x = ref.seeded_vector(m2.cols, 7)
    assert np.array_equal(spmv_scatter_baseline(to_dg(m2), x, 9).view(np.uint64),
                          ref.spmv_scatter(m2, x, 9, 2).view(np.uint64))


def test_scatter_more_chunks_than_columns(ref):
    m = ref.generate(prostate_desk())
    x = ref.seeded_vector(m.cols, 3)
    chunks = m.cols + 17
    assert np.array_equal(spmv_scatter_baseline(to_dg(m), x, chunks).view(np.uint64),
                          ref.spmv_scatter(m, x, chunks, 1).view(np.uint64))


def test_gather_beats_scatter_on_c2_sample():
    """The paper's comparison (the gather kernel 3-4x faster than the scatter
    GPU baseline), here on a 1M-row C2-profile sample."""
    import torch
    p = dg.profiles.c2(rows=1_000_000)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)  # our launches and the timing events on one real stream
    with dg.DoseEngine.generate(p) as e:
        m = e.copy_rows(0, p.rows)
        x = torch.from_numpy(dg.seeded_vector(p.cols, 42)).cuda()
        y = torch.empty(p.rows, dtype=torch.float64, device="cuda")

        def t(fn, n=5):
            fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(n):
                fn()
            b.record()
            torch.cuda.synchronize()
            return a.elapsed_time(b) / n

        g = t(lambda: e.dose_device(x.data_ptr(), p.cols, y.data_ptr(), stream=st.cuda_stream, sync=False))
    with ScatterEngine(m, 148) as s:
        sc = t(lambda: s.dose_device(x.data_ptr(), p.cols, y.data_ptr(), stream=st.cuda_stream))
    print(f"gather {g:.3f} ms, scatter {sc:.3f} ms, ratio {sc / g:.2f}")
    assert sc > 1.5 * g
