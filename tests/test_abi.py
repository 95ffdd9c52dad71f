"""CPU suite: the C-ABI library loads, exports exactly what include/dosegpu.h declares, and its
host-only logic (status strings, perf-model bytes, nnz-balanced partitioner, option checks)
behaves; on a box without a GPU every compute entry point fails loudly with DG_ERR_NO_DEVICE
instead of falling back to the CPU."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2103_09683_b200 as dg
from paper_2103_09683_b200 import dose as D

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "dosegpu.h")).read()
    return sorted(set(re.findall(r"\b(dg_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(D.LIB_PATH)
    declared = header_symbols()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), name
    # and the Python binding covers the whole declared surface
    assert set(declared) == set(dg.exported_symbols())


def test_library_is_sm100a_only():
    out = os.popen(f"cuobjdump --list-elf {D.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", ""))


def test_exact_kernels_have_no_fma():
    """-ffp-contract=off semantics (proj/CMakeLists.txt:10-12): the exact dose kernels must issue
    separate DMUL/DADD, never DFMA."""
    sass = os.popen(f"cuobjdump -sass {D.LIB_PATH} 2>&1").read()
    funcs = re.split(r"\n\s*Function : ", sass)
    exact = [f for f in funcs if re.match(r"\S*k_(warp|group|block)\w*_exact|\S*exact", f)]
    exact = [f for f in funcs if "exact" in f.split("\n", 1)[0]]
    assert exact, "no exact kernels found in SASS"
    for f in exact:
        name = f.split("\n", 1)[0]
        assert "DFMA" not in f, name
        assert "DMUL" in f and "DADD" in f, name


def test_strerror_matches_errc_names():
    lib = D._lib()
    names = [e.name for e in dg.Errc]
    for i, n in enumerate(names):
        assert lib.dg_strerror(i + 1).decode() == n
    assert lib.dg_strerror(0).decode() == "OK"
    assert lib.dg_strerror(900).decode() == "NoDevice"


def test_traffic_bytes_is_layout_of_model():
    """perf_model.cpp:41-54 with layout_of: (vb+ib)*nnz + 16*nr + 8*nc."""
    assert dg.traffic_bytes(1_000_000, 4096, 40_774_090) == 179_129_128
    assert dg.traffic_bytes(2_970_000, 68_000, 1_480_000_000, 2, 4) == \
        6 * 1_480_000_000 + 16 * 2_970_000 + 8 * 68_000


def _partition_ref(lens, bpn, parts):
    w = np.concatenate([[0], np.cumsum(np.asarray(lens, dtype=np.int64) * bpn + 16)])
    total = w[-1]
    b = [0]
    for g in range(1, parts):
        b.append(int(np.argmax(w * parts >= g * total)))
    b.append(len(lens))
    return np.array(b, dtype=np.uint64)


@pytest.mark.parametrize("parts", [1, 2, 3, 4, 8])
def test_partition_is_nnz_balanced(parts):
    rng = np.random.default_rng(parts)
    lens = np.where(rng.random(5000) < 0.7, 0, np.exp(rng.normal(5, 1.3, 5000)).astype(np.int64))
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    b = dg.partition_rows(rp, parts)
    assert np.array_equal(b, _partition_ref(lens, 4, parts))
    assert np.array_equal(b, dg.partition_lengths(lens.astype(np.uint32), parts))
    assert b[0] == 0 and b[-1] == len(lens) and np.all(np.diff(b.astype(np.int64)) >= 0)
    loads = [int((rp[b[g + 1]] - rp[b[g]]) * 4 + 16 * (b[g + 1] - b[g])) for g in range(parts)]
    assert max(loads) - min(loads) <= 2 * (4 * lens.max() + 16)


def test_partition_edge_cases():
    assert list(dg.partition_rows(np.zeros(1, dtype=np.uint64), 4)) == [0, 0, 0, 0, 0]
    b = dg.partition_rows(np.array([0, 100], dtype=np.uint64), 3)
    assert b[0] == 0 and b[-1] == 1
    with pytest.raises(dg.Error) as e:
        dg.partition_rows(np.array([0, 5, 3], dtype=np.uint64), 2)
    assert e.value.code == dg.Errc.ValidationFailure
    with pytest.raises(dg.Error):
        dg.partition_rows(np.array([0, 1], dtype=np.uint64), 0)


def test_default_options_struct():
    o = D._Options()
    D._lib().dg_default_options(C.byref(o))
    assert o.struct_size == C.sizeof(D._Options) == 32
    assert (o.device, o.lane_width, o.accumulation, o.row_begin, o.row_end) == (-1, 32, 0, 0, 0)


def _no_gpu():
    try:
        import torch
        return not torch.cuda.is_available()
    except Exception:
        return True


@pytest.mark.skipif(not _no_gpu(), reason="checks the no-GPU behaviour")
def test_no_device_fails_loudly(port):
    from oracle.oracle import liver_desk
    m = port.generate(liver_desk())
    cm = dg.CsrMatrix(m.rows, m.cols, m.index_width, m.row_ptr, m.col, m.values, m.precision)
    with pytest.raises(dg.Error) as e:
        dg.spmv_rowchunk(cm, np.zeros(m.cols))
    assert e.value.status == 900
    with pytest.raises(dg.Error):
        dg.DoseEngine.generate(dg.profiles.liver_desk())
    with pytest.raises(dg.Error) as e:  # the multi-device handle too
        dg.MultiDoseEngine.from_csr(cm, [0, 0])
    assert e.value.status == 900
    with pytest.raises(dg.Error) as e:
        dg.MultiDoseEngine.generate(dg.profiles.liver_desk(), [0])
    assert e.value.status == 900


def test_multi_options_and_status_codes():
    o = D._MultiOptions()
    D._lib().dg_multi_default_options(C.byref(o))
    assert o.struct_size == C.sizeof(D._MultiOptions) == 4 * (2 + 16 + 3)
    assert (o.n_devices, o.devices[0], o.lane_width, o.accumulation, o.gather) == \
        (1, 0, 32, 0, dg.GATHER_PEER)
    lib = D._lib()
    assert lib.dg_strerror(902).decode() == "NoNccl"
    assert lib.dg_strerror(2003).decode() == "NcclError"
    assert lib.dg_strerror(1002).decode() == "CudaError"
    # option errors come before any device work: a bad struct size is InvalidConfig
    o.struct_size = 4
    h = C.c_void_p()
    view = D._View()
    assert lib.dg_multi_create(C.byref(view), C.byref(o), C.byref(h)) == 1 + dg.Errc.InvalidConfig
    o.struct_size = C.sizeof(D._MultiOptions)
    o.n_devices = 0
    assert lib.dg_multi_create(C.byref(view), C.byref(o), C.byref(h)) == 1 + dg.Errc.InvalidConfig
    o.n_devices, o.gather = 1, 7
    assert lib.dg_multi_create(C.byref(view), C.byref(o), C.byref(h)) == 1 + dg.Errc.InvalidConfig


def test_out_array_is_checked():
    """DoseEngine.dose(out=...) hands out's pointer to the library: a wrong dtype, size or
    layout must raise instead of letting the library write past the buffer."""
    D._out_array(np.empty(5), 5)
    for bad in (np.empty(5, dtype=np.float32), np.empty(4), np.empty(10)[::2], np.empty(6)):
        with pytest.raises(ValueError):
            D._out_array(bad, 5)


@pytest.mark.parametrize("name", ["c1", "liver-desk", "prostate-desk"])
def test_seeded_vector_pinned_to_reference_golden(golden, name):
    """dg_seeded_vector (the headline bench's x) against the reference's own x: golden.json holds
    checksum_bits(ddm::seeded_vector(cols, 42)) written by the reference (make_golden.py;
    bench.cpp:31-36)."""
    cols = {"c1": 4096, "liver-desk": 6800, "prostate-desk": 5090}[name]
    assert f"{dg.checksum_bits(dg.seeded_vector(cols, 42)):016x}" == golden[name]["x_fnv"]


@pytest.mark.parametrize("n,seed", [(40_000, 42), (196_608, 1000), (196_608, 1099), (1, 0), (0, 7)])
def test_seeded_vector_equals_reference_at_config_sizes(ref, n, seed):
    """C2's x and C4's optimisation-loop x_k = seeded_vector(196608, 1000 + k), bit for bit against
    the reference compiled from its own sources (oracle/_ref)."""
    a = dg.seeded_vector(n, seed)
    b = ref.seeded_vector(n, seed)
    assert np.array_equal(a.view(np.uint64), np.asarray(b, dtype=np.float64).view(np.uint64))


@pytest.mark.parametrize("case", ["inconsistent", "ratio_above_1", "negative_sigma", "all_empty",
                                  "zero_ratio_not_empty", "window_above_cols", "consistent"])
def test_generator_profile_contract_matches_reference(case):
    """dg_create_generated / dg_generated_row_lengths check a profile exactly as
    ddm::validate_profile does (matgen.cpp:96-126): the same Errc in the same order -- ranges
    (InvalidConfig), then the length distribution's expected nnz ratio within 10% of the target
    (InconsistentProfile).  Profile errors come back before any device is touched (this runs on
    the CPU); a consistent profile gets as far as the device (NoDevice here)."""
    from oracle.oracle import Oracle, OracleError, Profile as OProfile, have_reference
    base = [5000, 4096, 0.01, 0.70, 4.5741, 0.8278, 4096, 1]  # C1's profile, fewer rows
    mod = {"inconsistent": (4, 5.5), "ratio_above_1": (2, 1.5), "negative_sigma": (5, -0.1),
           "all_empty": (3, 1.0), "zero_ratio_not_empty": (2, 0.0), "window_above_cols": (6, 5000),
           "consistent": None}[case]
    if mod:
        base[mod[0]] = mod[1]
    want = 0
    if have_reference():
        try:
            Oracle("reference").generate(OProfile(*base))
        except OracleError as e:
            want = e.code
    else:  # the reference's Errc for each case (matgen.cpp:96-126)
        want = {"inconsistent": 15, "all_empty": 15, "zero_ratio_not_empty": 15,
                "consistent": 0}.get(case, 6)
    with pytest.raises(dg.Error) as err:
        dg.generated_row_lengths(dg.Profile(*base), 0, 10)
    got = err.value.status
    if want == 0:
        assert got == 900  # NoDevice: the profile passed
    else:
        assert got == want, (case, got, want)
