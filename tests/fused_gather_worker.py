"""torchrun worker for tests/test_fused_gather_gpu.py::test_fused_gather_two_processes_ipc.

Each rank holds one nnz-balanced row shard of a generated matrix, registers every rank's full-d
buffer (its own + the peer's CUDA IPC mapping) as gather targets (argv[2] "epilogue": stores from
the dose kernels; "blocks": copy-engine copies per finished row block) and checks its full d against
the single-device dose bit for bit, over several doses with different x."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

import paper_2103_09683_b200 as dg
from paper_2103_09683_b200.sharded import ShardedDose


def main(out_dir: str, mode: str = "epilogue") -> None:
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    p = dg.profiles.c1()
    p.rows = 400_000
    sd = ShardedDose.for_generated(p, rank=rank, world=world, device=0)
    fg = sd.enable_fused_gather(mode=mode)
    y_local = torch.empty(sd.local_rows, dtype=torch.float64, device="cuda")
    with dg.DoseEngine.generate(p, device=0) as whole:
        for seed in (42, 5, 6):
            x_host = dg.seeded_vector(p.cols, seed)
            want = whole.dose(x_host)
            x = torch.from_numpy(x_host).cuda()
            full = fg.dose(x, y_local)
            got = full.cpu().numpy()
            assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (rank, seed)
            assert np.array_equal(y_local.cpu().numpy().view(np.uint64),
                                  want[sd.row_begin:sd.row_end].view(np.uint64))
            dist.barrier()  # nobody starts the next dose (re-zeroing) while a peer still reads
    sd.close()
    with open(os.path.join(out_dir, f"ok{rank}"), "w") as f:
        f.write("ok\n")
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1], *(sys.argv[2:3]))
