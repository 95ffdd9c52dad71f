"""The multi-device handle (dg_multi_*, include/dosegpu.h): one process, several GPUs behind one
call -- the reference's own fan-out (ddm::spmv_rowchunk -> parallel_blocks, spmv.hpp:37,
spmv.cpp:17-32) over devices.  The pool's boxes have one GPU, so the shards are virtual (the same
device listed several times) for the PEER / NONE gathers; NCCL needs distinct devices and runs
as a one-rank communicator here.  Bits must equal the one-device dose (rows are independent)."""
import ctypes as C

import numpy as np
import pytest

import paper_2103_09683_b200 as dg
from paper_2103_09683_b200 import dose as D
from oracle.oracle import c1_profile, liver_desk

pytestmark = pytest.mark.gpu


def bits(a):
    return np.asarray(a, dtype=np.float64).view(np.uint64)


def to_dg(m):
    return dg.CsrMatrix(m.rows, m.cols, m.index_width, m.row_ptr, m.col, m.values, m.precision)


@pytest.fixture(scope="module")
def liver(port):
    return port.generate(liver_desk())


def _device_array(ptr, n):
    import torch

    class _A:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False),
                                    "version": 2, "strides": None}
    return torch.as_tensor(_A(), device="cuda:0").cpu().numpy()


@pytest.mark.parametrize("gather", [dg.GATHER_NONE, dg.GATHER_PEER])
@pytest.mark.parametrize("n", [1, 2, 3, 8])
def test_virtual_shards_match_single_device(port, liver, gather, n):
    x = port.seeded_vector(liver.cols, 42)
    want = port.spmv_rowchunk(liver, x, 32, 4)
    with dg.MultiDoseEngine.from_csr(to_dg(liver), [0] * n, gather=gather) as m:
        assert m.n_shards == n and m.bounds[0] == 0 and m.bounds[-1] == liver.rows
        got = m.dose(x)
        assert np.array_equal(bits(got), bits(want))
        for i in range(n):
            full, sl = m.device_d(i)
            assert sl == full + 8 * int(m.bounds[i])
            d = _device_array(full, liver.rows)
            r0, r1 = int(m.bounds[i]), int(m.bounds[i + 1])
            assert np.array_equal(bits(d[r0:r1]), bits(want[r0:r1]))  # own slice always
            if gather == dg.GATHER_PEER:  # every device holds the full d
                assert np.array_equal(bits(d), bits(want))
        t = m.last_timing()
        assert t["ms_total"] > 0 and t["ms_kernels"] > 0


@pytest.mark.parametrize("blocks", ["4", "16"])
def test_peer_gather_overlapped_per_row_block(port, liver, monkeypatch, blocks):
    """PEER gather with row blocks: each shard's dose copies every block into the other devices'
    full d as soon as its tile kernel flags the block done, while later blocks are computed.  x
    changes every dose, so a block copied before its rows were final would hold the previous
    dose's values on some device."""
    import torch
    monkeypatch.setenv("DG_BLOCKS", blocks)
    monkeypatch.setenv("DG_SINK_OVERLAP", "1")  # (same-device sinks copy after the kernels otherwise)
    with dg.MultiDoseEngine.from_csr(to_dg(liver), [0, 0, 0], gather=dg.GATHER_PEER) as m:
        for seed in (5, 6, 7, 8):
            x = port.seeded_vector(liver.cols, seed)
            want = bits(port.spmv_rowchunk(liver, x, 32, 4))
            xd = torch.from_numpy(x).cuda()
            m.dose_device(xd.data_ptr(), xd.numel())
            for i in range(3):
                full, _ = m.device_d(i)
                assert np.array_equal(bits(_device_array(full, liver.rows)), want), (seed, i)
            assert np.array_equal(bits(m.dose(x)), want)


@pytest.mark.parametrize("gather", [dg.GATHER_NONE, dg.GATHER_PEER])
@pytest.mark.parametrize("blocks", ["1", "8"])
def test_pinned_host_d_downloaded_per_row_block(port, liver, monkeypatch, gather, blocks):
    """Pinned host d: each shard's dose downloads its slice row block by row block as its tile
    kernel finishes each block (over each device's own link).  x alternates, host d prefilled
    with NaN: every dose's host d equals the reference's bit for bit."""
    import torch
    monkeypatch.setenv("DG_BLOCKS", blocks)
    with dg.MultiDoseEngine.from_csr(to_dg(liver), [0, 0, 0], gather=gather) as m:
        yh = torch.full((liver.rows,), float("nan"), dtype=torch.float64).pin_memory()
        for seed in (11, 12, 13):
            x = port.seeded_vector(liver.cols, seed)
            xh = torch.from_numpy(x).pin_memory()
            m.dose_host_ptrs(xh.data_ptr(), liver.cols, yh.data_ptr())
            assert np.array_equal(bits(yh.numpy()), bits(port.spmv_rowchunk(liver, x, 32, 4))), seed
            if gather == dg.GATHER_PEER:
                for i in range(3):
                    full, _ = m.device_d(i)
                    assert np.array_equal(bits(_device_array(full, liver.rows)), bits(yh.numpy()))


def test_device_x_and_repeated_doses(port, liver):
    import torch
    with dg.MultiDoseEngine.from_csr(to_dg(liver), [0, 0, 0, 0]) as m:
        for seed in (1, 2, 3):
            x = port.seeded_vector(liver.cols, seed)
            xd = torch.from_numpy(x).cuda()
            m.dose_device(xd.data_ptr(), xd.numel())
            full, _ = m.device_d(2)
            assert np.array_equal(bits(_device_array(full, liver.rows)),
                                  bits(port.spmv_rowchunk(liver, x, 32, 4)))
        with pytest.raises(dg.Error) as e:
            m.dose(np.zeros(liver.cols + 1))
        assert e.value.code == dg.Errc.DimensionMismatch


def test_nccl_gather_one_rank_and_duplicate_devices(port, liver):
    x = port.seeded_vector(liver.cols, 42)
    want = port.spmv_rowchunk(liver, x, 32, 4)
    with pytest.raises(dg.Error) as e:  # one rank per GPU
        dg.MultiDoseEngine.from_csr(to_dg(liver), [0, 0], gather=dg.GATHER_NCCL)
    assert e.value.code == dg.Errc.InvalidConfig
    try:
        m = dg.MultiDoseEngine.from_csr(to_dg(liver), [0], gather=dg.GATHER_NCCL)
    except dg.Error as err:
        if err.status == 902:
            pytest.skip("libnccl.so.2 not loadable")
        raise
    with m:
        assert np.array_equal(bits(m.dose(x)), bits(want))


def test_generated_shards_and_fp32(port):
    p = dg.profiles.c1()
    p.rows = 200_000
    x = port.seeded_vector(p.cols, 42)
    with dg.DoseEngine.generate(p) as one:
        want = one.dose(x)
    with dg.MultiDoseEngine.generate(p, [0] * 4) as m:
        assert np.array_equal(bits(m.dose(x)), bits(want))
    with dg.MultiDoseEngine.generate(p, [0, 0], accumulation=dg.ACCUM_FP32) as m:
        gf = m.dose(x)
    assert np.max(np.abs(gf - want)) <= 1e-5 * np.max(np.abs(want))


def test_multi_config_errors(liver):
    with pytest.raises(dg.Error) as e:
        dg.MultiDoseEngine.from_csr(to_dg(liver), [0, 99])
    assert e.value.code == dg.Errc.InvalidConfig
    with pytest.raises(dg.Error) as e:
        dg.MultiDoseEngine.from_csr(to_dg(liver), [0], lane_width=3)
    assert e.value.code == dg.Errc.InvalidConfig
