#!/usr/bin/env python
"""Workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): small matrices
that drive every synchronisation mechanism of the dose kernels, each result checked against the
oracle so a run that 'passes' the sanitizer also computed the right bits.

  * desk matrices (liver / prostate): slice-stream tile kernel (TMA x windows, mbarrier ring,
    replicated windows), sub-warp bins, every lane width path, fp32 family;
  * _wide_row_matrix: wide sparse rows split into waves with carried partials (sNaN-flagged
    slots spin-waited on) in ONE fused launch, and k_dense;
  * a shard with DG_DENSE=1: k_dense followed by the tile kernel as a programmatic dependent
    launch;
  * host d with DG_BLOCKS=8: the overlapped download (row-block epoch flags released by the
    kernel, cuStreamWaitValue32 on the copy stream);
  * the multi-device handle on virtual shards (peer copies).

    compute-sanitizer --tool racecheck python scripts/sanitize_run.py [--quick]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2103_09683_b200 as dg  # noqa: E402
from oracle.oracle import Oracle, liver_desk, prostate_desk  # noqa: E402
from test_parity_gpu import _wide_row_matrix, bits, to_dg  # noqa: E402


def check(name, got, want):
    ok = np.array_equal(bits(got), bits(want))
    print(f"{name}: {'ok' if ok else 'MISMATCH'}", flush=True)
    if not ok:
        raise SystemExit(f"{name}: result differs from the oracle")


def main():
    quick = "--quick" in sys.argv
    port = Oracle("port")
    liver = port.generate(liver_desk())
    x = port.seeded_vector(liver.cols, 42)
    check("liver exact L=32", dg.spmv_rowchunk(to_dg(liver), x), port.spmv_rowchunk(liver, x, 32, 1))
    with dg.DoseEngine.from_csr(to_dg(liver), accumulation=dg.ACCUM_FP32) as e:
        y = e.dose(x)
        want = port.spmv_rowchunk(liver, x, 1, 1)
        assert np.max(np.abs(y - want)) <= 1e-5 * np.max(np.abs(want))
        print("liver fp32: ok", flush=True)
    if not quick:
        for L in (1, 4, 64):
            check(f"liver L={L}", dg.spmv_rowchunk(to_dg(liver), x, dg.RowChunkConfig(L)),
                  port.spmv_rowchunk(liver, x, L, 1))
        pro = port.generate(prostate_desk())
        xp = port.seeded_vector(pro.cols, 42)
        check("prostate exact", dg.spmv_rowchunk(to_dg(pro), xp), port.spmv_rowchunk(pro, xp, 32, 1))
    # split rows: carried partials, all waves in one launch; k_dense for the wide dense rows
    wide = _wide_row_matrix(port, rows=1500 if quick else 3000)
    xw = port.seeded_vector(wide.cols, 42)
    os.environ["DG_TILE_NNZ"] = "4096"
    with dg.DoseEngine.from_csr(to_dg(wide)) as e:
        check("wide rows fused waves (dose 1)", e.dose(xw), port.spmv_rowchunk(wide, xw, 32, 1))
        x2 = port.seeded_vector(wide.cols, 7)
        check("wide rows fused waves (dose 2)", e.dose(x2), port.spmv_rowchunk(wide, x2, 32, 1))
    del os.environ["DG_TILE_NNZ"]
    # k_dense -> tile kernel as a programmatic dependent launch (device x / y, no profiling)
    import torch
    os.environ["DG_DENSE"] = "1"
    nosplit = _wide_row_matrix(port, rows=1500, split=False, seed=9)
    xn = port.seeded_vector(nosplit.cols, 42)
    with dg.DoseEngine.from_csr(to_dg(nosplit)) as e:
        xd = torch.from_numpy(xn).cuda()
        yd = torch.empty(nosplit.rows, dtype=torch.float64, device="cuda")
        e.dose_device(xd.data_ptr(), nosplit.cols, yd.data_ptr())
        check("k_dense + PDL tile kernel", yd.cpu().numpy(), port.spmv_rowchunk(nosplit, xn, 32, 1))
    del os.environ["DG_DENSE"]
    # overlapped host download: row-block flags + cuStreamWaitValue32
    os.environ["DG_BLOCKS"] = "8"
    with dg.DoseEngine.from_csr(to_dg(liver)) as e:
        check("overlapped download", e.dose(x), port.spmv_rowchunk(liver, x, 32, 1))
    del os.environ["DG_BLOCKS"]
    # multi-device handle (virtual shards, peer copies)
    with dg.MultiDoseEngine.from_csr(to_dg(liver), [0, 0, 0]) as m:
        check("multi-device peer gather", m.dose(x), port.spmv_rowchunk(liver, x, 32, 1))
    print("sanitize_run: all ok", flush=True)


if __name__ == "__main__":
    main()
