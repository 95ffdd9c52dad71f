"""Randomised parity sweep (GPU): matrices mixing every row kind the planner distinguishes --
empty rows, short rows (<= 32), sparse rows in a locality window, contiguous rows (the value
stream), dense-but-gapped rows, rows spanning many windows (split into waves with carried
partials) -- at U16 and U32 widths, under several plan knobs.  Exact family: bits equal
ddm::spmv_rowchunk (the C oracle, lane width 32); fp32 family: within 1e-5 * max|d|.
Reference anchor: the lane-strided row semantics of src/spmv.cpp:48-68."""
import numpy as np
import pytest

import paper_2103_09683_b200 as dg
from oracle.oracle import HALF, U16, U32, Csr

pytestmark = pytest.mark.gpu
FP32_TOL = 1e-5


def _random_matrix(rng, rows, cols, iw):
    out = []
    for _ in range(rows):
        kind = rng.choice(["empty", "short", "sparse", "contig", "gapped", "wide"],
                          p=[0.35, 0.15, 0.25, 0.1, 0.1, 0.05])
        if kind == "empty":
            c = np.array([], dtype=np.int64)
        elif kind == "short":
            n = int(rng.integers(1, 33))
            c = np.sort(rng.choice(cols, n, replace=False))
        elif kind == "sparse":
            w = int(min(cols, rng.integers(64, 4097)))
            lo = int(rng.integers(0, cols - w + 1))
            n = int(rng.integers(33, max(34, w // 2)))
            c = lo + np.sort(rng.choice(w, min(n, w), replace=False))
        elif kind == "contig":
            n = int(min(cols, rng.integers(33, 9000)))
            lo = int(rng.integers(0, cols - n + 1))
            c = np.arange(lo, lo + n)
        elif kind == "gapped":  # >= 3/4 of its span, not contiguous
            n = int(min(cols - 1, rng.integers(100, 6000)))
            span = min(cols, n + max(1, n // 5))
            lo = int(rng.integers(0, cols - span + 1))
            c = lo + np.sort(rng.choice(span, n, replace=False))
        else:  # sparse over the whole width: several windows, carried partials
            n = int(rng.integers(200, 3000))
            c = np.sort(rng.choice(cols, min(n, cols), replace=False))
        out.append(c)
    lens = np.array([len(c) for c in out])
    rp = np.zeros(rows + 1, dtype=np.uint64)
    np.cumsum(lens, out=rp[1:])
    col = np.concatenate(out).astype(np.uint32) if len(out) else np.zeros(0, np.uint32)
    nnz = len(col)
    v = (rng.random(nnz) * (1 - 2.0 ** -14) + 2.0 ** -14)
    v[rng.random(nnz) < 0.1] *= -1  # some negative values
    return Csr(rows, cols, HALF, iw, rp, col, v.astype(np.float16).view(np.uint16))


@pytest.mark.parametrize("seed", range(24))
def test_random_matrices_bit_exact(port, monkeypatch, seed):
    rng = np.random.default_rng(1000 + seed)
    cols = [4096, 20_000, 65_535, 90_000][seed % 4]
    iw = U32 if cols >= 65_536 or seed % 3 == 0 else U16
    knobs = [{}, {"DG_DENSE_MIN_LEN": "64"}, {"DG_TILE_NNZ": "4096"},
             {"DG_DENSE_ORDER": "len", "DG_BLOCKS": "4"}][(seed // 4 + seed) % 4]
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    m = _random_matrix(rng, int(rng.integers(500, 2500)), cols, iw)
    x = rng.random(cols)
    want = port.spmv_rowchunk(m, x, 32, 2)
    csr = dg.CsrMatrix(m.rows, m.cols, m.index_width, m.row_ptr, m.col, m.values, m.precision)
    with dg.DoseEngine.from_csr(csr) as e:
        for _ in range(2):
            got = e.dose(x)
            assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (seed, knobs)
        back = e.copy_rows(0, m.rows)
        assert np.array_equal(back.col_indices, m.col)
        assert np.array_equal(back.values, m.values)
    with dg.DoseEngine.from_csr(csr, accumulation=dg.ACCUM_FP32) as e:
        got = e.dose(x)
        ref = port.spmv_oracle(m, x)
        assert np.max(np.abs(got - ref)) <= FP32_TOL * np.max(np.abs(ref)), (seed, knobs)
