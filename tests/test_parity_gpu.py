"""GPU parity suite: the CUDA dose path (through the C ABI) against the oracle and the
reference's golden vectors.  Exact family: bit-identical to ddm::spmv_rowchunk for the same
lane_width.  fp32 family: per-voxel |d - d_oracle| <= 1e-5 * max|d_oracle| (north_star)."""
import os

import numpy as np
import pytest

import paper_2103_09683_b200 as dg
from oracle.oracle import (DOUBLE, HALF, SINGLE, U16, U32, Csr, c1_profile, liver_desk,
                           prostate_desk)

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
PROFILES = {"liver-desk": liver_desk, "prostate-desk": prostate_desk}
FP32_TOL = 1e-5  # north_star: per-voxel error <= 1e-5 relative to max dose


def bits(a):
    return np.asarray(a, dtype=np.float64).view(np.uint64)


def to_dg(m: Csr) -> dg.CsrMatrix:
    return dg.CsrMatrix(m.rows, m.cols, m.index_width, m.row_ptr, m.col, m.values, m.precision)


def from_dg(m: dg.CsrMatrix) -> Csr:
    return Csr(m.rows, m.cols, m.precision, m.index_width, m.row_ptr, m.col_indices, m.values)


def make_csr(rows, cols, entries, prec=DOUBLE, port=None, iw=U32):
    entries = sorted(entries)
    rp = np.zeros(rows + 1, dtype=np.uint64)
    for r, _, _ in entries:
        rp[r + 1] += 1
    rp = np.cumsum(rp).astype(np.uint64)
    col = np.array([c for _, c, _ in entries], dtype=np.uint32)
    v = np.array([val for _, _, val in entries], dtype=np.float64)
    if prec == HALF:
        v = np.array([port.encode_half(a) for a in v], dtype=np.uint16)
    elif prec == SINGLE:
        v = v.astype(np.float32)
    return Csr(rows, cols, prec, iw, rp, col, v)


@pytest.fixture(scope="module")
def desk(port):
    return {n: port.generate(p()) for n, p in PROFILES.items()}


# ------------------------------------------------------------------ golden parity ----------
@pytest.mark.parametrize("name", ["liver-desk", "prostate-desk"])
def test_desk_every_lane_width_matches_reference(port, golden, desk, name):
    m = desk[name]
    x = port.seeded_vector(m.cols, 42)
    for L, ck in golden[name]["rowchunk"].items():
        y = dg.spmv_rowchunk(to_dg(m), x, dg.RowChunkConfig(int(L)))
        assert f"{dg.checksum_bits(y):016x}" == ck, f"lane_width {L}"
    y1 = dg.spmv_oracle(to_dg(m), x)
    assert f"{dg.checksum_bits(y1):016x}" == golden[name]["oracle"]


@pytest.mark.parametrize("name", ["liver-desk", "prostate-desk"])
def test_desk_precisions_match_reference(port, golden, name):
    for prec, ck in golden[name]["precision"].items():
        m = port.generate(PROFILES[name](), int(prec))
        x = port.seeded_vector(m.cols, 42)
        y = dg.spmv_rowchunk(to_dg(m), x)
        assert f"{dg.checksum_bits(y):016x}" == ck["rowchunk32"]
        assert f"{dg.checksum_bits(dg.spmv_oracle(to_dg(m), x)):016x}" == ck["oracle"]


@pytest.mark.parametrize("name", ["liver-desk", "prostate-desk"])
def test_acceptance_seeds_match_reference(port, golden, name):
    """acceptance.cpp:148-175 profiles x seeds 11..14 with x = seeded_vector(cols, seed+1000)."""
    for seed, ck in golden[name]["seeds"].items():
        p = PROFILES[name]()
        p.seed = int(seed)
        m = port.generate(p)
        x = port.seeded_vector(m.cols, int(seed) + 1000)
        assert f"{dg.checksum_bits(dg.spmv_rowchunk(to_dg(m), x)):016x}" == ck["rowchunk32"]


def test_c1_matches_reference(port, golden):
    """configs[0]: 1M x 4096, 40.8M nnz; d bit-identical to the reference's rowchunk{32}."""
    m = port.generate(c1_profile())
    x = port.seeded_vector(m.cols, 42)
    with dg.DoseEngine.from_csr(to_dg(m)) as e:
        for _ in range(3):  # run_bench's drift check (bench.cpp:72-78)
            y = e.dose(x)
            assert f"{dg.checksum_bits(y):016x}" == golden["c1"]["rowchunk"]["32"]
    with dg.DoseEngine.from_csr(to_dg(m), accumulation=dg.ACCUM_FP32) as e:
        yf = e.dose(x)
    want = port.spmv_oracle(m, x)
    assert np.max(np.abs(yf - want)) <= FP32_TOL * np.max(np.abs(want))


def test_index_decoding_round_trip(port, desk):
    """P1: bit-exact index/row decoding -- the device copy reads back identical arrays."""
    for m in desk.values():
        with dg.DoseEngine.from_csr(to_dg(m)) as e:
            back = e.copy_rows(0, m.rows)
            assert np.array_equal(back.row_ptr, m.row_ptr)
            assert np.array_equal(back.col_indices, m.col)
            assert np.array_equal(back.values, m.values)
            mid = e.copy_rows(1000, 2000)
            assert np.array_equal(mid.col_indices, m.col[m.row_ptr[1000]:m.row_ptr[2000]])


def test_fp32_family_within_tolerance(port, desk):
    for m in desk.values():
        x = port.seeded_vector(m.cols, 42)
        with dg.DoseEngine.from_csr(to_dg(m), accumulation=dg.ACCUM_FP32) as e:
            y = e.dose(x)
        want = port.spmv_oracle(m, x)
        err = np.max(np.abs(y - want)) / np.max(np.abs(want))
        assert err <= FP32_TOL, err
        assert np.all(bits(y[want == 0]) == 0)


# ------------------------------------------------------------------ reference KATs ----------
def test_kat_2x2_half(port):
    """test_spmv.cpp:55-60"""
    m = make_csr(2, 2, [(0, 0, 1.0), (0, 1, 2.0), (1, 1, 3.0)], HALF, port)
    assert list(dg.spmv_oracle(to_dg(m), np.ones(2))) == [3.0, 3.0]
    assert list(dg.spmv_rowchunk(to_dg(m), np.ones(2))) == [3.0, 3.0]


def test_kat_empty_rows_positive_zero(port):
    """test_spmv.cpp:62-71"""
    m = make_csr(4, 3, [])
    for L in (1, 32, 64):
        y = dg.spmv_rowchunk(to_dg(m), np.array([1.0, 2.0, 3.0]), dg.RowChunkConfig(L, 2))
        assert len(y) == 4 and np.all(bits(y) == 0)


def test_kat_identity_257(port):
    """test_spmv.cpp:73-84: identity(257) half * x == x bit-exact for L in {1, 8, 1024}."""
    n = 257
    m = make_csr(n, n, [(i, i, 1.0) for i in range(n)], HALF, port)
    x = 0.25 + np.arange(n, dtype=np.float64)
    for L in (1, 8, 32, 1024):
        assert np.array_equal(bits(dg.spmv_rowchunk(to_dg(m), x, dg.RowChunkConfig(L, 3))), bits(x))


def test_kat_all_ones_row():
    """test_spmv.cpp:86-95: 1x64 all-ones -> 64.0 for every L <= 64."""
    m = make_csr(1, 64, [(0, c, 1.0) for c in range(64)])
    L = 1
    while L <= 64:
        assert dg.spmv_rowchunk(to_dg(m), np.ones(64), dg.RowChunkConfig(L))[0] == 64.0
        L *= 2


def test_kat_pinned_tree():
    """test_spmv.cpp:104-121"""
    p = [1.0, -1.0 + 2.0 ** -53, -(2.0 ** -53), 2.0 ** -100]
    m = make_csr(1, 4, [(0, c, v) for c, v in enumerate(p)])
    y = dg.spmv_rowchunk(to_dg(m), np.ones(4), dg.RowChunkConfig(4))
    assert bits(y)[0] == 0 and y[0] != ((p[0] + p[1]) + p[2]) + p[3]
    # and the same row must also come out as +0.0 under the L = 32 short-row bins (G = 4)
    assert bits(dg.spmv_rowchunk(to_dg(m), np.ones(4)))[0] == 0


def test_kat_lane_assignment():
    """test_spmv.cpp:123-135"""
    m = make_csr(1, 4, [(0, 0, 1.0), (0, 1, -1.0), (0, 2, 1e-16), (0, 3, 3e-16)])
    y1 = dg.spmv_rowchunk(to_dg(m), np.ones(4), dg.RowChunkConfig(1))[0]
    y2 = dg.spmv_rowchunk(to_dg(m), np.ones(4), dg.RowChunkConfig(2))[0]
    assert y1 == ((1.0 + -1.0) + 1e-16) + 3e-16
    assert y2 == 3.0 * 2.0 ** -53


def test_kat_workers_never_change_bits(port, desk):
    """test_spmv.cpp:137-146: output bits independent of workers."""
    m = desk["liver-desk"]
    x = port.seeded_vector(m.cols, 42)
    ref = dg.spmv_rowchunk(to_dg(m), x, dg.RowChunkConfig(32, 1))
    for w in (2, 3, 8, 400):
        assert np.array_equal(bits(ref), bits(dg.spmv_rowchunk(to_dg(m), x, dg.RowChunkConfig(32, w))))


@pytest.mark.parametrize("prec", [HALF, SINGLE, DOUBLE])
def test_kat_integer_matrices(golden, prec):
    z = np.load(os.path.join(HERE, "golden", f"integer_{prec}.npz"))
    m = Csr(300, 120, prec, U32, z["row_ptr"], z["col"], z["values"])
    for L in (1, 2, 16, 32, 64, 128):
        y = dg.spmv_rowchunk(to_dg(m), z["x"], dg.RowChunkConfig(L, 3))
        assert np.array_equal(bits(y), bits(z["y"])), L


def test_kat_row_lengths_around_lane_width(port):
    """test_spmv.cpp:239-252 extended to L = 32's bins: rows of 0,1,7,8,9,29..33,64,65,257."""
    lengths = [0, 1, 2, 3, 4, 5, 7, 8, 9, 15, 16, 17, 29, 31, 32, 33, 63, 64, 65, 255, 256, 257, 1000]
    rng = np.random.default_rng(91)
    ents = []
    for r, n in enumerate(lengths):
        cs = np.sort(rng.choice(2048, n, replace=False))
        ents += [(r, int(c), float(rng.uniform(-1, 1))) for c in cs]
    for prec in (HALF, DOUBLE):
        m = make_csr(len(lengths), 2048, ents, prec, port)
        x = rng.uniform(-1, 1, 2048)
        for L in (1, 2, 4, 8, 16, 32, 64, 128, 512):
            want = port.spmv_rowchunk(m, x, L, 1)
            got = dg.spmv_rowchunk(to_dg(m), x, dg.RowChunkConfig(L))
            assert np.array_equal(bits(got), bits(want)), (prec, L)


def test_u16_storage_and_u32_storage_agree(port, desk):
    m = desk["prostate-desk"]
    x = port.seeded_vector(m.cols, 42)
    a = dg.spmv_rowchunk(to_dg(m), x)
    m16 = to_dg(m)
    m16.col_indices = m.col.astype(np.uint16)
    assert np.array_equal(bits(a), bits(dg.spmv_rowchunk(m16, x)))
    m32 = to_dg(m)
    m32.index_width = U32  # U32 tag: 4-byte device indices
    assert np.array_equal(bits(a), bits(dg.spmv_rowchunk(m32, x)))


# ------------------------------------------------------------------ error contract ---------
def test_config_errors(port):
    """test_spmv.cpp:156-171 error contract."""
    m = to_dg(make_csr(4, 4, [(i, i, 1.0) for i in range(4)]))
    for L in (0, 3, 48, 2048):
        with pytest.raises(dg.Error) as e:
            dg.spmv_rowchunk(m, np.ones(4), dg.RowChunkConfig(L, 1))
        assert e.value.code == dg.Errc.InvalidConfig, L
    with pytest.raises(dg.Error) as e:
        dg.spmv_rowchunk(m, np.ones(4), dg.RowChunkConfig(32, 0))
    assert e.value.code == dg.Errc.InvalidConfig
    with pytest.raises(dg.Error) as e:
        dg.spmv_rowchunk(m, np.ones(5))
    assert e.value.code == dg.Errc.DimensionMismatch
    with dg.DoseEngine.from_csr(m) as eng:
        with pytest.raises(dg.Error) as e:
            eng.dose(np.ones(3))
        assert e.value.code == dg.Errc.DimensionMismatch
    with pytest.raises(dg.Error) as e:
        dg.DoseEngine.from_csr(m, accumulation=dg.ACCUM_FP32, lane_width=8)
    assert e.value.code == dg.Errc.InvalidConfig


def test_validation_failures(port, desk):
    """ddm::validate invariants (sparse.cpp:197-255) enforced at upload."""
    base = desk["liver-desk"]
    lens = np.diff(base.row_ptr.astype(np.int64))
    r2 = int(np.nonzero(lens >= 2)[0][3])  # a row with at least two entries

    def broken(fn):
        m = Csr(base.rows, base.cols, base.precision, base.index_width, base.row_ptr.copy(),
                base.col.copy(), base.values.copy())
        fn(m)
        return to_dg(m)

    cases = {
        "col out of range": lambda m: m.col.__setitem__(int(m.row_ptr[r2]), m.cols),
        "unsorted cols": lambda m: m.col.__setitem__(slice(int(m.row_ptr[r2]), int(m.row_ptr[r2]) + 2),
                                                     m.col[int(m.row_ptr[r2]):int(m.row_ptr[r2]) + 2][::-1]),
        "duplicate col": lambda m: m.col.__setitem__(int(m.row_ptr[r2]) + 1, m.col[int(m.row_ptr[r2])]),
        "inf value": lambda m: m.values.__setitem__(12, 0x7C00),
        "nan value": lambda m: m.values.__setitem__(13, 0x7E00),
        "row_ptr decreasing": lambda m: m.row_ptr.__setitem__(r2, m.row_ptr[r2 + 1] + 1),
    }
    for what, fn in cases.items():
        m = broken(fn)
        with pytest.raises(dg.Error) as e:
            dg.DoseEngine.from_csr(m)
        assert e.value.code == dg.Errc.ValidationFailure, what
    wide = to_dg(make_csr(2, 70000, [(0, 69999, 1.0)]))
    wide.index_width = U16
    with pytest.raises(dg.Error) as e:
        dg.DoseEngine.from_csr(wide)
    assert e.value.code == dg.Errc.ValidationFailure


# ------------------------------------------------------------------ shards ------------------
@pytest.mark.parametrize("parts", [2, 4, 8])
def test_row_shards_compose_bit_identically(port, desk, parts):
    """8(e) determinism: G nnz-balanced shards (virtual GPUs on one device) concatenate to the
    single-GPU d bit for bit."""
    m = desk["prostate-desk"]
    x = port.seeded_vector(m.cols, 42)
    full = dg.spmv_rowchunk(to_dg(m), x)
    b = dg.partition_rows(m.row_ptr, parts)
    pieces = []
    for g in range(parts):
        with dg.DoseEngine.from_csr(to_dg(m), row_begin=int(b[g]), row_end=int(b[g + 1])) as e:
            assert e.info["rows"] == b[g + 1] - b[g]
            pieces.append(e.dose(x))
    assert np.array_equal(bits(np.concatenate(pieces)), bits(full))


# ------------------------------------------------------------------ device generator -------
def test_generator_shards_compose_and_are_deterministic():
    p = dg.profiles.c1()
    p.rows = 200_000
    with dg.DoseEngine.generate(p) as a, dg.DoseEngine.generate(p) as b:
        ma, mb = a.copy_rows(0, p.rows), b.copy_rows(0, p.rows)
        assert np.array_equal(ma.row_ptr, mb.row_ptr) and np.array_equal(ma.col_indices, mb.col_indices)
        assert np.array_equal(ma.values, mb.values)
    lens = dg.generated_row_lengths(p, 0, p.rows)
    assert np.array_equal(lens, np.diff(ma.row_ptr.astype(np.int64)))
    bnd = dg.partition_lengths(lens, 3)
    for g in range(3):
        with dg.DoseEngine.generate(p, row_begin=int(bnd[g]), row_end=int(bnd[g + 1])) as s:
            part = s.copy_rows(0, s.info["rows"])
            r0, r1 = int(bnd[g]), int(bnd[g + 1])
            assert np.array_equal(part.col_indices, ma.col_indices[ma.row_ptr[r0]:ma.row_ptr[r1]])
            assert np.array_equal(part.values, ma.values[ma.row_ptr[r0]:ma.row_ptr[r1]])


@pytest.mark.parametrize("which", ["liver-desk", "prostate-desk", "c1"])
def test_generator_statistics_match_profile(port, which):
    """acceptance.cpp:232-257: empty fraction 0.70 +- 0.01, nnz ratio within 10% of target,
    below-32 fraction near the reference generator's on the same profile."""
    p = dg.profiles.NAMED[which]()
    with dg.DoseEngine.generate(p) as e:
        m = e.copy_rows(0, p.rows)
    assert port.validate(from_dg(m)) == 0
    lens = np.diff(m.row_ptr.astype(np.int64))
    ref_m = port.generate(c1_profile() if which == "c1" else PROFILES[which]())
    ref_lens = np.diff(ref_m.row_ptr.astype(np.int64))
    assert abs(np.mean(lens == 0) - 0.70) <= 0.01
    ratio = m.nnz / (p.rows * p.cols)
    assert abs(ratio - p.target_nnz_ratio) / p.target_nnz_ratio <= 0.10
    ne, rne = lens[lens > 0], ref_lens[ref_lens > 0]
    assert abs(np.mean(ne < 32) - np.mean(rne < 32)) <= 0.02
    assert abs(np.mean(ne) - np.mean(rne)) / np.mean(rne) <= 0.05
    assert np.all(m.values >= 0x0400) and np.all(m.values <= 0x3C00)  # [2^-14, 1] in binary16


def test_generated_matrix_dose_matches_oracle(port):
    p = dg.profiles.prostate_desk()
    x = port.seeded_vector(p.cols, 42)
    with dg.DoseEngine.generate(p) as e:
        y = e.dose(x)
        m = from_dg(e.copy_rows(0, p.rows))
    assert np.array_equal(bits(y), bits(port.spmv_rowchunk(m, x, 32, 4)))


@pytest.mark.parametrize("fuse", ["1", "0"])
def test_multibeam_hstack_generator(port, monkeypatch, fuse):
    """C4 shape at small scale: 3 beams hstacked -> U32 indices, beam b's columns offset; rows
    span several beams, so they are split into waves (fused into one launch, or not)."""
    monkeypatch.setenv("DG_FUSE_WAVES", fuse)
    beams = [dg.Profile(20_000, 32_768, 0.0073, 0.70, 6.3386, 0.8278, 4096, 11 + b) for b in range(3)]
    with dg.DoseEngine.generate(beams) as e:
        assert e.info["cols"] == 3 * 32_768 and e.info["index_bytes"] == 4
        m = from_dg(e.copy_rows(0, 20_000))
        x = port.seeded_vector(m.cols, 1000)
        y = e.dose(x)
        # the optimisation loop: x changes every evaluation, host and device d
        import torch
        yd = torch.empty(20_000, dtype=torch.float64, device="cuda")
        for k in range(1, 4):
            xk = port.seeded_vector(m.cols, 1000 + k)
            want = bits(port.spmv_rowchunk(m, xk, 32, 4))
            assert np.array_equal(bits(e.dose(xk)), want), k
            e.dose_device(torch.from_numpy(xk).cuda().data_ptr(), m.cols, yd.data_ptr())
            assert np.array_equal(yd.cpu().numpy().view(np.uint64), want), k
    assert port.validate(m) == 0
    assert np.array_equal(bits(y), bits(port.spmv_rowchunk(m, x, 32, 4)))
    with dg.DoseEngine.generate(beams[1]) as single:
        m1 = from_dg(single.copy_rows(0, 20_000))
    # beam 1's block of the hstack is exactly beam 1's own matrix shifted by 32768
    sel = (m.col >= 32_768) & (m.col < 65_536)
    assert np.array_equal(m.col[sel] - 32_768, m1.col) and np.array_equal(m.values[sel], m1.values)


@pytest.mark.slow
def test_c2_full_scale_sampled_rows(port):
    """configs[1] at full size: 8M x 40k, ~3.2e9 nnz.  Rows are independent, so the oracle on a
    sampled sub-matrix is exact for those rows; plus repeat-run checksum stability."""
    x = port.seeded_vector(40_000, 42)
    with dg.DoseEngine.generate(dg.profiles.c2()) as e:
        assert e.info["nnz"] > 3.0e9
        y = e.dose(x)
        ck = dg.checksum_bits(y)
        assert dg.checksum_bits(e.dose(x)) == ck
        rng = np.random.default_rng(3)
        starts = np.sort(rng.choice(e.info["rows"] - 64, 24, replace=False))
        for s in starts:
            m = from_dg(e.copy_rows(int(s), int(s) + 64))
            want = port.spmv_rowchunk(m, x, 32, 1)
            assert np.array_equal(bits(y[s:s + 64]), bits(want))
        # the longest rows exercise the LPT-first warp bin
        lens = np.diff(e.row_ptr().astype(np.int64))
        for r in np.argsort(lens)[-8:]:
            m = from_dg(e.copy_rows(int(r), int(r) + 1))
            assert bits(y[r]) == bits(port.spmv_rowchunk(m, x, 32, 1))[0]


def _wide_row_matrix(port, rows=3000, cols=40_000, seed=5, split=True):
    """Sparse windowed rows + long dense rows wider than one shared-memory window + rows
    straddling window boundaries + (split=True) wide sparse rows, which are cut into multi-wave
    segments with carried lane partials."""
    rng = np.random.default_rng(seed)
    lens = np.where(rng.random(rows) < 0.5, 0, rng.integers(1, 3000, rows))
    lens[rng.choice(rows, 40, replace=False)] = rng.integers(14_000, cols + 1, 40)  # wide, dense
    lens[:3] = [cols, 13_823, 27_647]
    sparse_wide = rng.choice(np.arange(3, rows), 30 if split else 0, replace=False)
    lens[sparse_wide] = rng.integers(40, 3000, len(sparse_wide))
    rp = np.zeros(rows + 1, dtype=np.uint64)
    np.cumsum(lens, out=rp[1:])
    col = np.empty(int(rp[-1]), dtype=np.uint32)
    for r in range(rows):
        n = int(lens[r])
        if n == 0:
            continue
        if r in sparse_wide:  # spread over up to the whole column range
            c = np.sort(rng.choice(cols, n, replace=False))
        elif n >= 4096:
            lo = int(rng.integers(0, cols - n + 1))
            c = np.arange(lo, lo + n)
        else:
            lo = int(rng.integers(0, cols - 4096 + 1))
            c = np.sort(rng.choice(4096, n, replace=False)) + lo
        col[rp[r]:rp[r + 1]] = c
    vals = (rng.random(len(col)) * 0.999 + 2 ** -14).astype(np.float16).view(np.uint16)
    return Csr(rows, cols, HALF, U16, rp, col, vals)


@pytest.mark.parametrize("fuse", ["1", "0"])
@pytest.mark.parametrize("tile_nnz", ["4096", "262144"])
def test_windowed_tiles_with_split_rows_bit_exact(port, monkeypatch, tile_nnz, fuse):
    """Split rows carry lane partials between waves: in one launch (fused: per-row flags) or in
    one launch per wave."""
    monkeypatch.setenv("DG_TILE_NNZ", tile_nnz)
    monkeypatch.setenv("DG_FUSE_WAVES", fuse)
    m = _wide_row_matrix(port)
    x = port.seeded_vector(m.cols, 42)
    want = port.spmv_rowchunk(m, x, 32, 4)
    with dg.DoseEngine.from_csr(to_dg(m)) as e:
        got = e.dose(x)
        if fuse == "0":
            assert e.info["n_kernels"] >= 2  # >= 2 waves (sparse wide rows are split)
        # repeated doses: the fused plan's per-row flags are epoch-tagged, never stale
        for seed in (7, 8):
            x2 = port.seeded_vector(m.cols, seed)
            assert np.array_equal(bits(e.dose(x2)), bits(port.spmv_rowchunk(m, x2, 32, 4)))
    assert np.array_equal(bits(got), bits(want))
    for short_max in ("0", "32"):  # short rows folded into tiles / in sub-warp bins
        monkeypatch.setenv("DG_SHORT_MAX", short_max)
        with dg.DoseEngine.from_csr(to_dg(m)) as e:
            assert np.array_equal(bits(e.dose(x)), bits(want))
    with dg.DoseEngine.from_csr(to_dg(m), accumulation=dg.ACCUM_FP32) as e:
        gf = e.dose(x)
    assert np.max(np.abs(gf - want)) <= FP32_TOL * np.max(np.abs(want))


def test_u32_rows_spanning_a_million_columns_bit_exact(port, monkeypatch):
    """No limit on the segments of a row: U32 rows scattered over ~1M columns are cut into
    ~200 windowed segments (waves) carrying their lane partials (plan.cu returned
    UnsupportedFeature past 64).  Reference: rowchunk_rows handles every valid CsrMatrix
    (src/spmv.cpp:48-68)."""
    rng = np.random.default_rng(11)
    rows, cols = 1500, 1_000_003
    lens = np.where(rng.random(rows) < 0.4, 0, rng.integers(1, 600, rows))
    wide = rng.choice(rows, 25, replace=False)
    lens[wide] = rng.integers(2000, 9000, len(wide))
    lens[0] = 40_000  # a dense row wider than a window
    rp = np.zeros(rows + 1, dtype=np.uint64)
    np.cumsum(lens, out=rp[1:])
    col = np.empty(int(rp[-1]), dtype=np.uint32)
    for r in range(rows):
        n = int(lens[r])
        if n == 0:
            continue
        if r in wide:
            c = np.sort(rng.choice(cols, n, replace=False))
        elif r == 0:
            c = np.arange(500_000, 500_000 + n)
        else:
            lo = int(rng.integers(0, cols - 4096))
            c = np.sort(rng.choice(4096, n, replace=False)) + lo
        col[rp[r]:rp[r + 1]] = c
    vals = (rng.random(len(col)) * 0.999 + 2 ** -14).astype(np.float16).view(np.uint16)
    m = Csr(rows, cols, HALF, U32, rp, col, vals)
    x = port.seeded_vector(cols, 42)
    want = port.spmv_rowchunk(m, x, 32, 4)
    for fuse in ("1", "0"):  # DG_FUSE_WAVES=0 is overridden past 64 waves (one fused launch)
        monkeypatch.setenv("DG_FUSE_WAVES", fuse)
        with dg.DoseEngine.from_csr(to_dg(m)) as e:
            assert np.array_equal(bits(e.dose(x)), bits(want))
            x2 = port.seeded_vector(cols, 9)
            assert np.array_equal(bits(e.dose(x2)), bits(port.spmv_rowchunk(m, x2, 32, 4)))
    with dg.DoseEngine.from_csr(to_dg(m), accumulation=dg.ACCUM_FP32) as e:
        gf = e.dose(x)
    assert np.max(np.abs(gf - want)) <= FP32_TOL * np.max(np.abs(want))


@pytest.mark.parametrize("env", [{}, {"DG_DENSE": "1"}, {"DG_DENSE": "0"},
                                 {"DG_DENSE": "1", "DG_DENSE_MIN_LEN": "1024"}])
def test_dense_rows_kernel_bit_exact(port, monkeypatch, env):
    """Dense rows (>= 3/4 of their span, >= DG_DENSE_MIN_LEN long) go to k_dense, launched
    before the tile kernel, and must give the same bits as the reference, for device and host d
    (the host path downloads row blocks as the tile kernel completes them), over repeated
    doses."""
    import torch
    monkeypatch.setenv("DG_BLOCKS", "8")  # 8 output row blocks: the overlapped host download
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    m = _wide_row_matrix(port, rows=6000, split=False)
    with dg.DoseEngine.from_csr(to_dg(m)) as e:
        yd = torch.empty(m.rows, dtype=torch.float64, device="cuda")
        for seed in (42, 7, 8):
            x = port.seeded_vector(m.cols, seed)
            want = bits(port.spmv_rowchunk(m, x, 32, 4))
            assert np.array_equal(bits(e.dose(x)), want), seed
            e.dose_device(torch.from_numpy(x).cuda().data_ptr(), m.cols, yd.data_ptr())
            assert np.array_equal(yd.cpu().numpy().view(np.uint64), want), seed
    with dg.DoseEngine.from_csr(to_dg(m), accumulation=dg.ACCUM_FP32) as e:
        x = port.seeded_vector(m.cols, 42)
        want = port.spmv_rowchunk(m, x, 32, 4)
        assert np.max(np.abs(e.dose(x) - want)) <= FP32_TOL * np.max(np.abs(want))


def test_small_tiles_desk_bit_exact(port, golden, desk, monkeypatch):
    monkeypatch.setenv("DG_TILE_NNZ", "2048")
    for name in ("liver-desk", "prostate-desk"):
        m = desk[name]
        x = port.seeded_vector(m.cols, 42)
        y = dg.spmv_rowchunk(to_dg(m), x)
        assert f"{dg.checksum_bits(y):016x}" == golden[name]["rowchunk"]["32"]


def test_v0_warp_plan_still_bit_exact(port, golden, desk, monkeypatch):
    """DG_PLAN=warp selects the v0 warp-per-row plan (kept for A/B measurement)."""
    monkeypatch.setenv("DG_PLAN", "warp")
    m = desk["prostate-desk"]
    x = port.seeded_vector(m.cols, 42)
    assert f"{dg.checksum_bits(dg.spmv_rowchunk(to_dg(m), x)):016x}" == \
        golden["prostate-desk"]["rowchunk"]["32"]


def test_overlapped_download_matches_device_result(monkeypatch):
    """Host d is downloaded block by block as the tile kernel publishes row-block completion
    (cuStreamWaitValue32 on per-block epochs); repeated doses must never read a stale block."""
    import torch
    p = dg.profiles.c1()
    with dg.DoseEngine.generate(p) as e:
        assert e.info["nnz"] > 16 << 20  # large enough for 8 output row blocks
        yd = torch.empty(p.rows, dtype=torch.float64, device="cuda")
        for seed in (42, 7, 8, 9):
            x = dg.seeded_vector(p.cols, seed)
            xd = torch.from_numpy(x).cuda()
            e.dose_device(xd.data_ptr(), p.cols, yd.data_ptr())
            yh = e.dose(x)  # overlapped path
            assert np.array_equal(bits(yh), yd.cpu().numpy().view(np.uint64)), seed
    monkeypatch.setenv("DG_NO_OVERLAP", "1")
    with dg.DoseEngine.generate(p) as e:
        assert np.array_equal(bits(e.dose(x)), bits(yh))


def _edge_values(rng, n):
    """binary16 bit patterns: both signs, subnormals, normals up to the largest finite."""
    v = rng.choice([0x0001, 0x03FF, 0x0400, 0x3C00, 0x7BFF, 0x8001, 0xBC00, 0xFBFF], n)
    mix = rng.random(n) < 0.7
    v[mix] = (rng.random(mix.sum()) * 2 - 1).astype(np.float16).view(np.uint16)[:mix.sum()]
    return v.astype(np.uint16)


@pytest.mark.parametrize("dense", ["0", "1"])
def test_edge_max_u16_width_and_special_values(port, monkeypatch, dense):
    """cols = 65535 (the widest U16 matrix): a fully dense 65535-long row (k_dense or global-x
    tiles), rows touching columns 0 and 65534, sparse rows over the whole width (split into
    waves), value bits with both signs / subnormals / the largest finite half, and an x with
    negatives, subnormals, -0.0 and magnitudes up to 1e290 (no sum overflows: an Inf - Inf NaN's
    payload is platform-defined)."""
    monkeypatch.setenv("DG_DENSE", dense)
    rng = np.random.default_rng(11)
    cols = 65_535
    rows_cols = [np.arange(cols), np.array([0, cols - 1]), np.array([cols - 1]), np.array([0])]
    for _ in range(200):
        n = int(rng.integers(1, 5000))
        rows_cols.append(np.sort(rng.choice(cols, n, replace=False)))
    for _ in range(100):
        rows_cols.append(np.array([], dtype=np.int64))
    rng.shuffle(rows_cols)
    lens = np.array([len(c) for c in rows_cols])
    rp = np.zeros(len(rows_cols) + 1, dtype=np.uint64)
    np.cumsum(lens, out=rp[1:])
    col = np.concatenate(rows_cols).astype(np.uint32)
    m = Csr(len(rows_cols), cols, HALF, U16, rp, col, _edge_values(rng, len(col)))
    x = rng.standard_normal(cols) * np.exp(rng.uniform(-700, 668, cols))  # no sum overflows
    x[rng.choice(cols, 50, replace=False)] = -0.0
    x[rng.choice(cols, 50, replace=False)] = 5e-324
    want = port.spmv_rowchunk(m, x, 32, 2)
    with dg.DoseEngine.from_csr(to_dg(m)) as e:
        assert np.array_equal(bits(e.dose(x)), bits(want))


def test_edge_odd_cols_unaligned_x(port):
    """cols not a multiple of 2 (x rows are staged into the padded buffer for TMA) and x passed
    from an unaligned device address."""
    import torch
    rng = np.random.default_rng(4)
    cols = 4095
    entries = [(r, int(c), float(rng.random()))
               for r in range(600) for c in rng.choice(cols, int(rng.integers(0, 300)), replace=False)]
    m = make_csr(600, cols, entries, HALF, port, U16)
    x = port.seeded_vector(cols, 42)
    want = bits(port.spmv_rowchunk(m, x, 32, 2))
    with dg.DoseEngine.from_csr(to_dg(m)) as e:
        assert np.array_equal(bits(e.dose(x)), want)
        buf = torch.zeros(cols + 1, dtype=torch.float64, device="cuda")
        buf[1:] = torch.from_numpy(x).cuda()
        y = torch.empty(600, dtype=torch.float64, device="cuda")
        e.dose_device(buf[1:].data_ptr(), cols, y.data_ptr())  # 8-byte, not 16-byte aligned
        assert np.array_equal(y.cpu().numpy().view(np.uint64), want)


def test_edge_no_rows_no_nonzeros(port):
    """rows = 0, and rows > 0 with nnz = 0 (every row empty: +0.0)."""
    m0 = make_csr(0, 3, [], HALF, port, U16)
    assert len(dg.spmv_rowchunk(to_dg(m0), np.ones(3))) == 0
    m1 = make_csr(5, 7, [], HALF, port, U16)
    y = dg.spmv_rowchunk(to_dg(m1), np.arange(7, dtype=np.float64))
    assert len(y) == 5 and np.all(bits(y) == 0)


@pytest.mark.parametrize("short", ["0", "1"])
def test_batch_width_both_paths_desk(port, golden, desk, monkeypatch, short):
    """4-chunk batches (short segments, chosen automatically when the mean segment is < 256
    nonzeros) and 8-chunk batches give the reference's bits on both desk profiles and C1-like
    rows."""
    monkeypatch.setenv("DG_SHORT_SEGMENTS", short)
    for name in ("liver-desk", "prostate-desk"):
        m = desk[name]
        x = port.seeded_vector(m.cols, 42)
        y = dg.spmv_rowchunk(to_dg(m), x)
        assert f"{dg.checksum_bits(y):016x}" == golden[name]["rowchunk"]["32"], name
    m = _wide_row_matrix(port, rows=2000, split=False)
    x = port.seeded_vector(m.cols, 42)
    assert np.array_equal(bits(dg.spmv_rowchunk(to_dg(m), x)), bits(port.spmv_rowchunk(m, x, 32, 2)))


@pytest.mark.parametrize("min_len", ["4096", "64"])
@pytest.mark.parametrize("iw", [U16, U32])
def test_contiguous_rows_values_only_bit_exact(port, monkeypatch, min_len, iw):
    """Contiguous rows (columns lo .. lo + len - 1) of at least DG_DENSE_MIN_LEN go to
    k_dense_values as binary16 values alone (the column is lo + position).  Rows start at column
    0 and end at the last column, have lengths around the 256-position batch edges, and end right
    before 'poison' columns that no row touches, where x is +Inf or NaN: a padding position that
    read x past the row's end (instead of the staged +0.0) would turn the row into NaN.  Exact
    family bit-identical to the reference (device and host d, repeated doses); fp32 family within
    tolerance; the device copy decodes back to the same arrays."""
    import torch
    monkeypatch.setenv("DG_DENSE_MIN_LEN", min_len)
    monkeypatch.setenv("DG_BLOCKS", "4")  # the overlapped host download
    rng = np.random.default_rng(21)
    cols = 20_000
    poison = np.array([5000, 10_000, 15_000])
    rows_cols = []
    ok = np.setdiff1d(np.arange(cols), poison)
    for p in poison:  # contiguous rows ending right before / starting right after a poison column
        for n in (64, 255, 256, 257, 4096, 4097, 4999):
            rows_cols.append(np.arange(p - n, p))
            rows_cols.append(np.arange(p + 1, min(cols, p + 1 + n)))
    rows_cols += [np.arange(0, 4100), np.arange(cols - 4600, cols), np.arange(0, 4999)]
    for _ in range(150):  # contiguous rows of random lengths inside a poison-free span
        n = int(rng.integers(32, 4999))
        seg = int(rng.integers(0, 4))
        lo0, hi0 = (0, 5000) if seg == 0 else (poison[seg - 1] + 1, poison[seg] if seg < 3 else cols)
        if hi0 - lo0 > n:
            lo = int(rng.integers(lo0, hi0 - n))
            rows_cols.append(np.arange(lo, lo + n))
    for _ in range(150):  # sparse rows avoiding the poison columns
        n = int(rng.integers(1, 3000))
        rows_cols.append(np.sort(rng.choice(ok, n, replace=False)))
    rows_cols += [np.array([], dtype=np.int64)] * 40
    rng.shuffle(rows_cols)
    lens = np.array([len(c) for c in rows_cols])
    rp = np.zeros(len(rows_cols) + 1, dtype=np.uint64)
    np.cumsum(lens, out=rp[1:])
    col = np.concatenate(rows_cols).astype(np.uint32)
    m = Csr(len(rows_cols), cols, HALF, iw, rp, col, _edge_values(rng, len(col)))
    x = rng.standard_normal(cols) * np.exp(rng.uniform(-20, 20, cols))
    x[poison] = [np.inf, np.nan, -np.inf]
    want = bits(port.spmv_rowchunk(m, x, 32, 2))
    assert not np.isnan(want.view(np.float64)).any()
    with dg.DoseEngine.from_csr(to_dg(m)) as e:
        yd = torch.empty(m.rows, dtype=torch.float64, device="cuda")
        xh = torch.from_numpy(x).pin_memory()
        yh = torch.full((m.rows,), 7.0, dtype=torch.float64).pin_memory()
        for _ in range(2):
            assert np.array_equal(bits(e.dose(x)), want)  # pageable host d
            e.dose_device(torch.from_numpy(x).cuda().data_ptr(), m.cols, yd.data_ptr())
            assert np.array_equal(yd.cpu().numpy().view(np.uint64), want)
            # pinned host d: row blocks downloaded while the tile kernel runs
            e.dose_host_ptrs(xh.data_ptr(), m.cols, yh.data_ptr())
            assert np.array_equal(yh.numpy().view(np.uint64), want)
            yh.fill_(7.0)
        # alternating x on the pinned path: a block downloaded before its last tile finished
        # would keep the previous dose's values
        x2 = x * 2.0
        want2 = bits(port.spmv_rowchunk(m, x2, 32, 2))
        x2h = torch.from_numpy(x2).pin_memory()
        for it in range(6):
            xx, ww = (xh, want) if it % 2 == 0 else (x2h, want2)
            e.dose_host_ptrs(xx.data_ptr(), m.cols, yh.data_ptr())
            assert np.array_equal(yh.numpy().view(np.uint64), ww)
        back = e.copy_rows(0, m.rows)
        assert np.array_equal(back.row_ptr, m.row_ptr)
        assert np.array_equal(back.col_indices, m.col)
        assert np.array_equal(back.values, m.values)
    # fp32 family on the dose data's value ranges (positive halves, x in [0, 1)) with the same
    # poison columns: tolerance against the oracle
    vpos = (rng.random(len(col)) * (1 - 2.0 ** -14) + 2.0 ** -14).astype(np.float16).view(np.uint16)
    mp = Csr(m.rows, cols, HALF, iw, rp, col, vpos)
    xp = rng.random(cols)
    xp[poison] = np.inf
    ref = port.spmv_rowchunk(mp, xp, 32, 2)
    with dg.DoseEngine.from_csr(to_dg(mp), accumulation=dg.ACCUM_FP32) as e:
        got = e.dose(xp)
        assert np.max(np.abs(got - ref)) <= FP32_TOL * np.max(np.abs(ref))
