"""Parity at BASELINE.json's full sizes through size-independent properties (rows are
independent, so the oracle on sampled rows is exact for those rows; sharded and unsharded plans
must agree bit for bit; one launch per wave and one launch for all waves must agree bit for bit).

C2 = configs[1] (8M x 40k, 3.2e9 nnz), C3 = C2 in G row shards (configs[2]), C4 = configs[3]
(6-beam hstack, U32 indices, multi-wave rows), C5 = one GPU's share of a configs[4] scenario."""
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


def test_c5_gpu_share_sampled_rows(port):
    """One GPU's 1/8 of a C5 scenario (88M x 40k rows overall): 11M rows, ~4.4e9 nnz."""
    p = dg.profiles.c5_scenarios()[0]
    lens = dg.generated_row_lengths(p, 0, p.rows)
    b = dg.partition_lengths(lens, 8, 4)
    x = dg.seeded_vector(p.cols, 42)
    with dg.DoseEngine.generate(p, row_begin=int(b[3]), row_end=int(b[4])) as e:
        assert e.info["nnz"] > 4.0e9
        y = e.dose(x)
        _sampled_rows_match(port, e, x, y)
