"""Parity at BASELINE.json's full sizes through size-independent properties (rows are
independent, so the oracle on sampled rows is exact for those rows; sharded and unsharded plans
must agree bit for bit; one launch per wave and one launch for all waves must agree bit for bit).

C2 = configs[1] (8M x 40k, 3.2e9 nnz), C3 = C2 in G row shards (configs[2]), C4 = configs[3]
(6-beam hstack, U32 indices, multi-wave rows), C5 = one GPU's share of a configs[4] scenario."""
import os

import numpy as np
import pytest

import paper_2103_09683_b200 as dg
from test_parity_gpu import bits, from_dg

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _sampled_rows_match(port, e, x, y, n_blocks=12, block=32, longest=6, seed=3):
    rng = np.random.default_rng(seed)
    rows = e.info["rows"]
    for s in np.sort(rng.choice(rows - block, n_blocks, replace=False)):
        m = from_dg(e.copy_rows(int(s), int(s) + block))
        assert np.array_equal(bits(y[s:s + block]), bits(port.spmv_rowchunk(m, x, 32, 1))), s
    lens = np.diff(e.row_ptr().astype(np.int64))
    for r in np.argsort(lens)[-longest:]:  # the longest rows (k_dense / global x / most waves)
        m = from_dg(e.copy_rows(int(r), int(r) + 1))
        assert bits(y[r]) == bits(port.spmv_rowchunk(m, x, 32, 1))[0], r


def _full_vector_match(port, e, x, y, y_fp32=None, block_nnz=300_000_000):
    """EVERY row of d against the C oracle: the resident matrix is copied back to the host in
    row blocks (dg_copy_rows, the reference's encoding) and each block is evaluated by the oracle
    on all host threads.  Exact family: bit-identical to rowchunk L=32 (src/spmv.cpp:48-68).
    y_fp32 (optional): the fp32 family's d, checked per voxel against spmv_oracle (= rowchunk
    L=1, bit for bit: test_spmv.cpp:97-102) within 1e-5 * max|d_oracle| (north_star).
    Returns (max|d_oracle|, max fp32 error)."""
    workers = os.cpu_count() or 1
    rp = e.row_ptr().astype(np.int64)
    rows = e.info["rows"]
    max_d = max_err = 0.0
    r0 = 0
    while r0 < rows:
        r1 = int(np.searchsorted(rp, rp[r0] + block_nnz, side="right")) - 1
        r1 = min(rows, max(r1, r0 + 1))
        m = from_dg(e.copy_rows(r0, r1))
        want = port.spmv_rowchunk(m, x, 32, workers)
        got = y[r0:r1]
        if not np.array_equal(bits(got), bits(want)):
            bad = np.nonzero(bits(got) != bits(want))[0]
            raise AssertionError(f"{len(bad)} rows differ in [{r0}, {r1}), first {r0 + bad[0]}")
        if y_fp32 is not None:
            ref1 = port.spmv_rowchunk(m, x, 1, workers)
            max_d = max(max_d, float(np.max(np.abs(ref1))) if len(ref1) else 0.0)
            if len(ref1):
                max_err = max(max_err, float(np.max(np.abs(y_fp32[r0:r1] - ref1))))
        r0 = r1
    return max_d, max_err


def test_c2_full_vector_exact_and_fp32(port):
    """configs[1] at full size (8M x 40k, 3.18e9 nnz): all 8M rows of the exact d bit-identical
    to the oracle's rowchunk L=32, and all 8M rows of the fp32 family within 1e-5 * max|d|."""
    p = dg.profiles.c2()
    x = dg.seeded_vector(p.cols, 42)
    with dg.DoseEngine.generate(p, accumulation=dg.ACCUM_FP32) as ef:
        y32 = ef.dose(x)
    with dg.DoseEngine.generate(p) as e:
        assert e.info["nnz"] > 3.0e9
        y = e.dose(x)
        max_d, max_err = _full_vector_match(port, e, x, y, y32)
    assert max_err <= 1e-5 * max_d, (max_err, max_d)
    print(f"C2 fp32 family: max error {max_err / max_d:.3e} of max|d|")


def test_c4_full_vector_exact(port):
    """configs[3] at full size (6-beam hstack, 2.97M x 196,608, U32, ~4.3e9 nnz, rows split into
    waves with carried partials): every row bit-identical to the oracle, for two x of the
    optimisation loop."""
    ps = dg.profiles.c4_beams()
    cols = sum(p.cols for p in ps)
    with dg.DoseEngine.generate(ps) as e:
        for k in (0, 1):
            x = dg.seeded_vector(cols, 1000 + k)
            _full_vector_match(port, e, x, e.dose(x))


@pytest.mark.parametrize("blocks", ["16", "64"])
def test_c2_pinned_host_path_alternating_x(monkeypatch, blocks):
    """The end-to-end path bench.py times: pinned host x and d, each row block downloaded as soon
    as the tile kernel flags its last tile done (cuStreamWaitValue32), while later blocks are still
    computed.  x alternates between doses, so a block downloaded before its rows were final would
    show the previous dose's values; every dose's host d is bit-identical to the device-resident d
    of the same x (itself pinned to the oracle by test_c2_full_vector_exact_and_fp32)."""
    import torch
    monkeypatch.setenv("DG_BLOCKS", blocks)
    p = dg.profiles.c2()
    xs = [dg.seeded_vector(p.cols, 42), dg.seeded_vector(p.cols, 43)]
    with dg.DoseEngine.generate(p) as e:
        want = []
        for x in xs:
            yd = torch.empty(p.rows, dtype=torch.float64, device="cuda")
            e.dose_device(torch.from_numpy(x).cuda().data_ptr(), p.cols, yd.data_ptr())
            want.append(yd.cpu())
        xh = [torch.from_numpy(x).pin_memory() for x in xs]
        yh = torch.full((p.rows,), 7.0, dtype=torch.float64).pin_memory()
        for it in range(8):
            e.dose_host_ptrs(xh[it % 2].data_ptr(), p.cols, yh.data_ptr())
            assert torch.equal(yh.view(torch.int64), want[it % 2].view(torch.int64)), it


@pytest.mark.parametrize("G", [8])
def test_c3_shards_concatenate_to_the_single_gpu_dose(G):
    """Each rank's nnz-balanced row shard of C2 (exactly what bench.py --gpus G gives it; the
    small shards use k_dense, the full matrix does not) reproduces its slice of the 1-GPU d."""
    import torch
    p = dg.profiles.c2()
    x = torch.from_numpy(dg.seeded_vector(p.cols, 42)).cuda()
    with dg.DoseEngine.generate(p) as e:
        full = torch.empty(p.rows, dtype=torch.float64, device="cuda")
        e.dose_device(x.data_ptr(), p.cols, full.data_ptr())
    lens = dg.generated_row_lengths(p, 0, p.rows)
    b = dg.partition_lengths(lens, G, 4)
    for g in range(G):
        r0, r1 = int(b[g]), int(b[g + 1])
        with dg.DoseEngine.generate(p, row_begin=r0, row_end=r1) as e:
            y = torch.empty(r1 - r0, dtype=torch.float64, device="cuda")
            e.dose_device(x.data_ptr(), p.cols, y.data_ptr())
            assert torch.equal(y.view(torch.int64), full[r0:r1].view(torch.int64)), g


def test_c4_full_scale_fused_waves_and_sampled_rows(port, monkeypatch):
    """C4 rows span several beams: split into waves with carried partials.  All waves in one
    launch and one launch per wave give the same bits; sampled rows match the oracle."""
    ps = dg.profiles.c4_beams()
    cols = sum(p.cols for p in ps)
    x = dg.seeded_vector(cols, 1000)
    with dg.DoseEngine.generate(ps) as e:
        assert e.info["index_bytes"] == 4
        y = e.dose(x)
        assert dg.checksum_bits(e.dose(x)) == dg.checksum_bits(y)
        _sampled_rows_match(port, e, x, y)
    monkeypatch.setenv("DG_FUSE_WAVES", "0")
    with dg.DoseEngine.generate(ps) as e:
        assert np.array_equal(bits(e.dose(x)), bits(y))


def test_c5_gpu_share_full_vector(port):
    """One GPU's 1/8 of a C5 scenario (88M x 40k rows overall): 11M rows, ~4.4e9 nnz."""
    p = dg.profiles.c5_scenarios()[0]
    lens = dg.generated_row_lengths(p, 0, p.rows)
    b = dg.partition_lengths(lens, 8, 4)
    x = dg.seeded_vector(p.cols, 42)
    with dg.DoseEngine.generate(p, row_begin=int(b[3]), row_end=int(b[4])) as e:
        assert e.info["nnz"] > 4.0e9
        y = e.dose(x)
        _full_vector_match(port, e, x, y)  # all 11M rows
