"""N>1 path on CPU (gloo, world_size 2): nnz-balanced row sharding + the dose all-gather compose
into the single-device d bit for bit.  The per-shard compute here is the oracle (test
infrastructure), standing in for the per-GPU DoseEngine the B200 path uses; the partitioner
(libdosegpu.so host logic) and the collective (paper_2103_09683_b200/sharded.py) are the
product code under test."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, profile_name, out_q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_2103_09683_b200.sharded import ShardedDose, shard_bounds_from_row_ptr

        orc = O.Oracle("port")
        m = orc.generate(getattr(O, profile_name)())
        x = orc.seeded_vector(m.cols, 42)
        bounds = shard_bounds_from_row_ptr(m.row_ptr, world)

        def local(xt, yt):
            sub = m.take_rows(np.arange(int(bounds[rank]), int(bounds[rank + 1])))
            yt.copy_(torch.from_numpy(orc.spmv_rowchunk(sub, xt.numpy(), 32, 1)))

        sd = ShardedDose(None, rank=rank, world=world, device=-1, bounds=bounds, local=local)
        y_local = torch.empty(sd.local_rows, dtype=torch.float64)
        full = sd.dose(torch.from_numpy(x), y_local, gather=True)
        want = orc.spmv_rowchunk(m, x, 32, 1)
        ok = np.array_equal(full.numpy().view(np.uint64), want.view(np.uint64))
        nnz = [int(m.row_ptr[bounds[g + 1]] - m.row_ptr[bounds[g]]) for g in range(world)]
        out_q.put((rank, ok, nnz, [int(b) for b in bounds]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("profile_name", ["liver_desk", "prostate_desk"])
def test_row_sharded_dose_gathers_bit_identically(profile_name):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, profile_name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, nnz, bounds in res:
        assert ok, f"rank {rank}: gathered d differs from the single-device oracle"
        assert bounds[0] == 0 and bounds[-1] > bounds[1] > 0
        # nnz-balanced: shards within one max-row of each other
        assert abs(nnz[0] - nnz[1]) <= 0.02 * sum(nnz) + 10_000
