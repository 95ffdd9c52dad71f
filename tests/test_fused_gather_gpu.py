"""Fused d gather: the dose kernels store each finished row, at its global row
index, into every registered full-d buffer (dg_set_gather_targets).  Every target must equal the
single-device d bit for bit, whatever the kernel family that finished the row.

Single process: the "ranks" are shard engines on one device and the targets plain device buffers.
Two processes: real CUDA IPC mappings (dg_ipc_*) exchanged over a gloo group, both ranks on
cuda:0 -- the multi-GPU layout on a one-GPU box."""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2103_09683_b200 as dg
from test_parity_gpu import FP32_TOL, _wide_row_matrix, bits, to_dg

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _fused(m, x, parts, n_targets=2, **kw):
    """Shard engines [b_g, b_g+1) each storing into n_targets NaN-prefilled full-d buffers."""
    import torch
    targets = [torch.full((m.rows,), float("nan"), dtype=torch.float64, device="cuda")
               for _ in range(n_targets)]
    b = dg.partition_rows(m.row_ptr, parts)
    locals_ = []
    for g in range(parts):
        with dg.DoseEngine.from_csr(to_dg(m), row_begin=int(b[g]), row_end=int(b[g + 1]), **kw) as e:
            e.set_gather_targets([t.data_ptr() for t in targets])
            locals_.append(e.dose(x))
            e.set_gather_targets([])
    torch.cuda.synchronize()
    return [t.cpu().numpy() for t in targets], np.concatenate(locals_)


@pytest.mark.parametrize("lane_width", [1, 8, 32, 64, 256])
def test_fused_targets_bit_exact_every_lane_width(port, lane_width):
    m = _wide_row_matrix(port, rows=1500)
    x = port.seeded_vector(m.cols, 42)
    want = port.spmv_rowchunk(m, x, lane_width, 4)
    targets, local = _fused(m, x, 3, lane_width=lane_width)
    assert np.array_equal(bits(local), bits(want))
    for t in targets:
        assert np.array_equal(bits(t), bits(want))  # empty rows zero-filled (+0.0), not NaN


@pytest.mark.parametrize("env", [{}, {"DG_TILE_NNZ": "4096"}, {"DG_SHORT_MAX": "0"},
                                 {"DG_PLAN": "warp"}])
def test_fused_targets_every_plan(port, monkeypatch, env):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    m = _wide_row_matrix(port)
    x = port.seeded_vector(m.cols, 7)
    want = port.spmv_rowchunk(m, x, 32, 4)
    targets, _ = _fused(m, x, 2, n_targets=8)
    for t in targets:
        assert np.array_equal(bits(t), bits(want))


def test_fused_targets_fp32_family(port):
    m = _wide_row_matrix(port)
    x = port.seeded_vector(m.cols, 42)
    want = port.spmv_rowchunk(m, x, 32, 4)
    targets, local = _fused(m, x, 4, accumulation=dg.ACCUM_FP32)
    assert np.max(np.abs(local - want)) <= FP32_TOL * np.max(np.abs(want))
    for t in targets:
        assert np.array_equal(bits(t), bits(local))


def test_fused_targets_repeat_doses_and_generated_shards():
    """Repeated doses overwrite (the shard's range is re-zeroed each dose); generated shards."""
    import torch
    p = dg.profiles.c1()
    p.rows = 300_000
    with dg.DoseEngine.generate(p) as whole:
        lens = dg.generated_row_lengths(p, 0, p.rows)
        b = dg.partition_lengths(lens, 2)
        full = torch.full((p.rows,), float("nan"), dtype=torch.float64, device="cuda")
        shards = [dg.DoseEngine.generate(p, row_begin=int(b[g]), row_end=int(b[g + 1]))
                  for g in range(2)]
        for s in shards:
            s.set_gather_targets([full.data_ptr()])
        for seed in (42, 3):
            x = dg.seeded_vector(p.cols, seed)
            want = whole.dose(x)
            for s in shards:
                s.dose(x)
            assert np.array_equal(full.cpu().numpy().view(np.uint64), bits(want)), seed
        for s in shards:
            s.close()


def test_gather_target_errors():
    import torch
    m = dg.CsrMatrix(4, 4, dg.U16, np.array([0, 1, 1, 2, 2], dtype=np.uint64),
                     np.array([0, 3], dtype=np.uint32), np.array([0x3C00, 0x3C00], dtype=np.uint16))
    buf = torch.zeros(4, dtype=torch.float64, device="cuda")
    with dg.DoseEngine.from_csr(m) as e:
        with pytest.raises(dg.Error) as ei:
            e.set_gather_targets([buf.data_ptr()] * 9)  # more than kMaxGatherTargets
        assert ei.value.code == dg.Errc.InvalidConfig
        with pytest.raises(dg.Error):
            e.set_gather_targets([buf.data_ptr(), 0])
        e.set_gather_targets([buf.data_ptr()])
        e.dose(np.ones(4))
        assert buf.cpu().tolist() == [1.0, 0.0, 1.0, 0.0]


@pytest.mark.parametrize("lane_width", [1, 8, 32, 64])
def test_block_targets_every_lane_width(port, monkeypatch, lane_width):
    """Block targets on plans without row blocks (lane widths != 32, split rows): the shard's d
    is copied after its kernels; every target equals the reference's d bit for bit."""
    import torch
    monkeypatch.setenv("DG_BLOCKS", "4")
    m = _wide_row_matrix(port, rows=1500)
    x = port.seeded_vector(m.cols, 42)
    want = port.spmv_rowchunk(m, x, lane_width, 4)
    targets = [torch.full((m.rows,), float("nan"), dtype=torch.float64, device="cuda")
               for _ in range(2)]
    b = dg.partition_rows(m.row_ptr, 3)
    for g in range(3):
        with dg.DoseEngine.from_csr(to_dg(m), row_begin=int(b[g]), row_end=int(b[g + 1]),
                                    lane_width=lane_width) as e:
            e.set_block_targets([t.data_ptr() for t in targets])
            e.dose(x)
    torch.cuda.synchronize()
    for t in targets:
        assert np.array_equal(bits(t.cpu().numpy()), bits(want))


@pytest.mark.parametrize("blocks", ["4", "16"])
def test_block_targets_bit_exact_host_and_device_d(monkeypatch, blocks):
    """dg_set_block_targets: the shards' doses copy each finished row block into every full-d
    buffer (copy engines, started by the tile kernel's block flags).  Device-resident and host d,
    x alternating, NaN-prefilled targets: every target equals the single-device d bit for bit."""
    import torch
    monkeypatch.setenv("DG_BLOCKS", blocks)
    p = dg.profiles.c1()
    p.rows = 300_000
    with dg.DoseEngine.generate(p) as whole:
        lens = dg.generated_row_lengths(p, 0, p.rows)
        b = dg.partition_lengths(lens, 3)
        fulls = [torch.full((p.rows,), float("nan"), dtype=torch.float64, device="cuda")
                 for _ in range(2)]
        shards = [dg.DoseEngine.generate(p, row_begin=int(b[g]), row_end=int(b[g + 1]))
                  for g in range(3)]
        for s in shards:
            s.set_block_targets([f.data_ptr() for f in fulls])
        for it, seed in enumerate((42, 3, 4, 5)):
            x = dg.seeded_vector(p.cols, seed)
            want = bits(whole.dose(x))
            xd = torch.from_numpy(x).cuda()
            for g, s in enumerate(shards):
                if it % 2:
                    s.dose(x)  # host d
                else:
                    y = torch.empty(int(b[g + 1] - b[g]), dtype=torch.float64, device="cuda")
                    s.dose_device(xd.data_ptr(), p.cols, y.data_ptr())
            torch.cuda.synchronize()
            for f in fulls:
                assert np.array_equal(f.cpu().numpy().view(np.uint64), want), seed
        for s in shards:
            s.set_block_targets([])
            s.close()


@pytest.mark.parametrize("mode", ["epilogue", "blocks"])
def test_fused_gather_two_processes_ipc(tmp_path, mode):
    """Two ranks (gloo, both on cuda:0): IPC-mapped full-d buffers, each rank's kernels (mode
    "epilogue") or copy engines (mode "blocks") writing into the other's.  The worker asserts
    bit-equality with the single-device d."""
    env = dict(os.environ, PYTHONPATH=ROOT)
    if mode == "blocks":
        env["DG_BLOCKS"] = "8"  # several row blocks per shard: copies overlapped with the tiles
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29613" if mode == "epilogue" else "29614",
           os.path.join(ROOT, "tests", "fused_gather_worker.py"), str(tmp_path), mode]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    for g in range(2):
        assert (tmp_path / f"ok{g}").read_text().strip() == "ok"
