"""CPU suite: pin the oracle (C restatement, oracle/ddm_oracle.c) against the reference's golden
vectors (tests/golden, produced by the reference itself) and, where it is built, against the
reference library directly.  Re-expresses the reference's own KATs (proj/tests/test_spmv.cpp,
test_half.cpp, acceptance.cpp) as assertions on the oracle."""
import os

import numpy as np
import pytest

from oracle.oracle import (DOUBLE, HALF, SINGLE, U32, Csr, Profile, c1_profile, liver_desk,
                           prostate_desk, traffic_bytes)

HERE = os.path.dirname(os.path.abspath(__file__))
PROFILES = {"liver-desk": liver_desk, "prostate-desk": prostate_desk}


def fnv(port, b: bytes) -> str:
    import ctypes as C
    port.lib.or_fnv1a64.restype = C.c_uint64
    port.lib.or_fnv1a64.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64]
    return f"{port.lib.or_fnv1a64(b, len(b), 14695981039346656037):016x}"


def make_csr(rows, cols, entries, prec=DOUBLE, port=None):
    """test_helpers.hpp:17-26 make_csr: canonical row-major CSR from (r, c, v) triples."""
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
    return Csr(rows, cols, prec, U32, rp, col, v)


def bits(a):
    return np.asarray(a, dtype=np.float64).view(np.uint64)


# ------------------------------------------------------------------ golden pins -----------
@pytest.mark.parametrize("name", ["liver-desk", "prostate-desk"])
def test_generate_matches_golden(port, golden, name):
    m = port.generate(PROFILES[name]())
    g = golden[name]
    assert (m.rows, m.cols, m.nnz, m.index_width) == (g["rows"], g["cols"], g["nnz"], g["index_width"])
    assert fnv(port, m.values.tobytes()) == g["values_fnv"]
    assert fnv(port, m.col.tobytes()) == g["col_fnv"]
    assert fnv(port, m.row_ptr.tobytes()) == g["row_ptr_fnv"]
    assert port.validate(m) == 0


@pytest.mark.parametrize("name", ["liver-desk", "prostate-desk"])
def test_spmv_matches_golden_every_lane_width(port, golden, name):
    m = port.generate(PROFILES[name]())
    x = port.seeded_vector(m.cols, 42)
    g = golden[name]
    assert f"{port.checksum_bits(x):016x}" == g["x_fnv"]
    yo = port.spmv_oracle(m, x)
    assert f"{port.checksum_bits(yo):016x}" == g["oracle"]
    assert np.abs(yo).max() == g["max_abs"]
    for L, ck in g["rowchunk"].items():
        y = port.spmv_rowchunk(m, x, int(L), 4)
        assert f"{port.checksum_bits(y):016x}" == ck, L


@pytest.mark.parametrize("name", ["liver-desk", "prostate-desk"])
def test_precisions_and_seeds_match_golden(port, golden, name):
    g = golden[name]
    for prec, ck in g["precision"].items():
        m = port.generate(PROFILES[name](), int(prec))
        x = port.seeded_vector(m.cols, 42)
        assert f"{port.checksum_bits(port.spmv_rowchunk(m, x, 32, 2)):016x}" == ck["rowchunk32"]
        assert f"{port.checksum_bits(port.spmv_oracle(m, x)):016x}" == ck["oracle"]
    for seed, ck in g["seeds"].items():
        p = PROFILES[name]()
        p.seed = int(seed)
        m = port.generate(p)
        x = port.seeded_vector(m.cols, int(seed) + 1000)
        assert m.nnz == ck["nnz"]
        assert f"{port.checksum_bits(port.spmv_rowchunk(m, x, 32, 3)):016x}" == ck["rowchunk32"]
        assert f"{port.checksum_bits(port.spmv_oracle(m, x)):016x}" == ck["oracle"]


def test_c1_matches_golden(port, golden):
    """The BASELINE oracle config (1M x 4096, 40.8M nnz) reproduces the reference's checksums."""
    m = port.generate(c1_profile())
    g = golden["c1"]
    assert m.nnz == g["nnz"]
    assert fnv(port, m.values.tobytes()) == g["values_fnv"]
    x = port.seeded_vector(m.cols, 42)
    assert f"{port.checksum_bits(port.spmv_rowchunk(m, x, 32, 8)):016x}" == g["rowchunk"]["32"]
    assert f"{port.checksum_bits(port.spmv_rowchunk(m, x, 1, 8)):016x}" == g["oracle"]


def test_half_codec_matches_golden(port, golden):
    dec = np.array([port.decode_half(b) for b in range(65536)])
    keep = ~np.isnan(dec)
    assert fnv(port, dec[keep].tobytes()) == golden["half_decode_fnv"]
    z = np.load(os.path.join(HERE, "golden", "half_sweep.npz"))
    enc = np.array([port.encode_half(float(v)) for v in z["x"]], dtype=np.uint16)
    assert np.array_equal(enc, z["bits"])


def test_half_codec_kats(port):
    """test_half.cpp:64-80 decode KATs; acceptance.cpp:204-214 encode(decode(h)) == h."""
    assert port.decode_half(0x3C00) == 1.0 and port.decode_half(0xC000) == -2.0
    assert port.decode_half(0x7BFF) == 65504.0 and port.decode_half(0x0001) == 2.0 ** -24
    assert port.decode_half(0x03FF) == 2.0 ** -14 - 2.0 ** -24
    assert port.decode_half(0x3555) == 0.333251953125
    assert np.signbit(port.decode_half(0x8000))
    for b in range(0, 0x7C00, 7):
        assert port.encode_half(port.decode_half(b)) == b
    assert port.encode_half(65519.99) == 0x7BFF and port.encode_half(65520.0) == 0x7C00


@pytest.mark.parametrize("prec", [HALF, SINGLE, DOUBLE])
def test_integer_matrices_bit_exact(port, golden, prec):
    """acceptance.cpp:177-200: integer matrices make every lane width bit-exact."""
    z = np.load(os.path.join(HERE, "golden", f"integer_{prec}.npz"))
    m = Csr(300, 120, prec, U32, z["row_ptr"], z["col"], z["values"])
    for L in (1, 2, 16, 32, 64, 128):
        y = port.spmv_rowchunk(m, z["x"], L, 3)
        assert np.array_equal(bits(y), bits(z["y"]))
        assert f"{port.checksum_bits(y):016x}" == golden["integer"][str(prec)]["y"]


# ------------------------------------------------------------------ reference KATs ----------
def test_pinned_tree_kat(port):
    """test_spmv.cpp:104-121: (p0+p2)+(p1+p3) == 0.0 while the sequential sum is 2^-100."""
    p = [1.0, -1.0 + 2.0 ** -53, -(2.0 ** -53), 2.0 ** -100]
    m = make_csr(1, 4, [(0, c, v) for c, v in enumerate(p)])
    y = port.spmv_rowchunk(m, np.ones(4), 4, 1)
    assert bits(y)[0] == bits([0.0])[0]


def test_lane_assignment_kat(port):
    """test_spmv.cpp:123-135: L=1 vs L=2 differ; L=2 gives exactly 3*2^-53."""
    m = make_csr(1, 4, [(0, 0, 1.0), (0, 1, -1.0), (0, 2, 1e-16), (0, 3, 3e-16)])
    y1 = port.spmv_rowchunk(m, np.ones(4), 1, 1)[0]
    y2 = port.spmv_rowchunk(m, np.ones(4), 2, 1)[0]
    assert y1 == ((1.0 + -1.0) + 1e-16) + 3e-16
    assert y2 == 3.0 * 2.0 ** -53 and y1 != y2


def test_empty_rows_are_positive_zero(port):
    m = make_csr(4, 3, [])
    for L in (1, 32):
        y = port.spmv_rowchunk(m, np.array([1.0, 2.0, 3.0]), L, 2)
        assert np.all(bits(y) == 0)


def test_config_errors(port):
    """test_spmv.cpp:156-171: bad lane widths / workers -> InvalidConfig, x length -> DimMismatch."""
    from oracle.oracle import OracleError
    m = make_csr(4, 4, [(i, i, 1.0) for i in range(4)])
    for L in (0, 3, 48, 2048):
        with pytest.raises(OracleError) as e:
            port.spmv_rowchunk(m, np.ones(4), L, 1)
        assert e.value.code == 1 + 5
    with pytest.raises(OracleError) as e:
        port.spmv_rowchunk(m, np.ones(5), 32, 1)
    assert e.value.code == 1 + 4


def test_traffic_identity():
    """acceptance.cpp:84-100 (6nnz+12nr+8nc under the 4-byte row_ptr layout) and the layout_of
    form used as the roofline numerator."""
    rng = np.random.default_rng(123)
    for _ in range(200):
        nr, nc = int(rng.integers(1, 4_000_000)), int(rng.integers(1, 80_000))
        nnz = int(rng.integers(0, min(nr * nc, 2_000_000_000)))
        assert traffic_bytes(nr, nc, nnz) == 4 * nnz + 16 * nr + 8 * nc
        assert traffic_bytes(nr, nc, nnz, 2, 4) == 6 * nnz + 16 * nr + 8 * nc


# ------------------------------------------------------------------ port vs reference -------
def test_port_equals_reference_random_profiles(port, ref):
    rng = np.random.default_rng(5)
    for k in range(6):
        cols = int(rng.integers(64, 9000))
        win = int(rng.integers(1, cols + 1))
        sigma = float(rng.uniform(0.2, 1.4))
        ratio = 0.02
        mean_len = ratio * cols / 0.3
        mu = float(np.log(max(mean_len, 1.5)) - sigma ** 2 / 2)
        prof = Profile(int(rng.integers(100, 3000)), cols, ratio, 0.7, mu, sigma, win, 100 + k)
        for prec in (HALF, SINGLE):
            try:
                a = port.generate(prof, prec)
            except Exception as e:  # inconsistent profile: both must refuse identically
                with pytest.raises(type(e)):
                    ref.generate(prof, prec)
                continue
            b = ref.generate(prof, prec)
            assert np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col, b.col)
            assert np.array_equal(a.values, b.values)
            x = port.seeded_vector(a.cols, 7 + k)
            for L in (1, 8, 32, 64):
                assert np.array_equal(bits(port.spmv_rowchunk(a, x, L, 3)),
                                      bits(ref.spmv_rowchunk(b, x, L, 3)))


def test_port_validate_matches_reference(port, ref):
    m = port.generate(liver_desk())
    assert port.validate(m) == 0 == ref.validate(m)
    bad = Csr(m.rows, m.cols, m.precision, m.index_width, m.row_ptr.copy(), m.col.copy(),
              m.values.copy())
    bad.col[5] = bad.cols  # out of range
    assert port.validate(bad) != 0 and ref.validate(bad) != 0
    bad = Csr(m.rows, m.cols, m.precision, m.index_width, m.row_ptr.copy(), m.col.copy(),
              m.values.copy())
    bad.values[9] = 0x7C00  # +inf
    assert port.validate(bad) != 0 and ref.validate(bad) != 0
