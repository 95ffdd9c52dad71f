"""Row-sharded dose evaluation across GPUs (one process per GPU, torch.distributed plumbing).

SURVEY.md 8(e): rows are independent (``ddm::rowchunk_rows`` keeps no cross-row state,
src/spmv.cpp:53-67), so the matrix is cut into nnz-balanced contiguous row blocks
(``dg_partition_lengths``), each GPU holds its block plus a replicated x, and the only collective
is an all-gather of the dose slices -- used only when the full d must be resident on a device.
Output bits are identical for any number of GPUs (the row plan is per-row).

The d slices are unequal; ``gather_dose`` is an allgatherv made of one broadcast per shard into
place (NCCL on B200s, gloo in the CPU tests).
"""
from __future__ import annotations

from typing import Callable, Optional, Sequence

import numpy as np

from .dose import (ACCUM_EXACT, DoseEngine, generated_row_lengths, partition_lengths,
                   partition_rows)


def shard_bounds_from_lengths(lengths: np.ndarray, world: int, bytes_per_nnz: int = 4) -> np.ndarray:
    """bounds[g]..bounds[g+1] = rows of rank g (balanced on (vb+ib)*len + 16 bytes per row)."""
    return partition_lengths(lengths, world, bytes_per_nnz)


def shard_bounds_from_row_ptr(row_ptr: np.ndarray, world: int, bytes_per_nnz: int = 4) -> np.ndarray:
    return partition_rows(row_ptr, world, bytes_per_nnz)


CUDA_STREAM_LEGACY = 1  # cudaStreamLegacy: the legacy default stream as an explicit handle


def _torch_stream(device: int) -> int:
    """torch's current stream on `device` as a handle for dg_dose.  Torch's default stream is the
    legacy stream, whose handle is 0 -- which dg_dose reads as "the handle's own stream" -- so it
    is passed as cudaStreamLegacy instead."""
    import torch
    return torch.cuda.current_stream(device).cuda_stream or CUDA_STREAM_LEGACY


def gather_dose(y_local, bounds: Sequence[int], group=None, out=None):
    """Allgatherv of the unequal d slices into the full d on every rank (torch tensors on
    y_local's device): this rank's slice is copied into place, then one broadcast per shard g
    (root g) writes rows [bounds[g], bounds[g+1]) of every rank's full d directly -- no padding,
    no compaction.  The broadcasts are issued one after another (async, then
    waited): plain collectives every backend supports (the in-process C-ABI path, dg_multi,
    groups them into one NCCL call)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    me = dist.get_rank(group)
    n = int(bounds[world])
    full = out if out is not None else torch.empty(n, dtype=y_local.dtype, device=y_local.device)
    full[int(bounds[me]):int(bounds[me + 1])].copy_(y_local)
    works = []
    for g in range(world):
        if bounds[g + 1] > bounds[g]:
            src = dist.get_global_rank(group, g) if group is not None else g
            works.append(dist.broadcast(full[int(bounds[g]):int(bounds[g + 1])], src=src,
                                        group=group, async_op=True))
    for w in works:
        w.wait()
    return full


class ShardedDose:
    """This rank's shard of a row-partitioned matrix on its GPU.

    ``local``: a callable (x_device_tensor, y_device_tensor) -> None computing this rank's slice;
    by default a DoseEngine over the shard generated on the device.
    """

    def __init__(self, profiles, *, rank: int, world: int, device: int, bounds: np.ndarray,
                 accumulation: int = ACCUM_EXACT,
                 local: Optional[Callable] = None):
        self.rank, self.world, self.device = rank, world, device
        self.bounds = np.asarray(bounds, dtype=np.uint64)
        self.row_begin, self.row_end = int(self.bounds[rank]), int(self.bounds[rank + 1])
        self.engine = None
        if local is None:
            self.engine = DoseEngine.generate(profiles, row_begin=self.row_begin,
                                              row_end=self.row_end, device=device,
                                              accumulation=accumulation)
            self.local = self._engine_local
        else:
            self.local = local

    @classmethod
    def for_generated(cls, profiles, *, rank: int, world: int, device: int, **kw) -> "ShardedDose":
        ps = [profiles] if not isinstance(profiles, (list, tuple)) else list(profiles)
        cols = sum(p.cols for p in ps)
        lens = generated_row_lengths(ps, 0, ps[0].rows, device=device)
        bounds = shard_bounds_from_lengths(lens, world, 2 + (2 if cols < 65536 else 4))
        return cls(ps, rank=rank, world=world, device=device, bounds=bounds, **kw)

    def _engine_local(self, x, y, stream: int = 0):
        # default: torch's current stream on this device, so the dose is ordered after the torch
        # work that produced x and before the torch work (all-gather, copies) that reads y
        # (the handle's private stream would be ordered with neither -- ADVICE r01)
        if not stream:
            stream = _torch_stream(self.device)
        self.engine.dose_device(x.data_ptr(), x.numel(), y.data_ptr(), stream=stream, sync=False)

    @property
    def local_rows(self) -> int:
        return self.row_end - self.row_begin

    def dose(self, x, y_local, *, gather: bool = False, group=None, stream: int = 0):
        """Local slice into y_local; with gather=True also returns the full d (all-gather)."""
        if self.engine is not None:
            self.local(x, y_local, stream)
        else:
            self.local(x, y_local)
        if gather:
            return gather_dose(y_local, self.bounds, group)
        return None

    def enable_fused_gather(self, group=None, mode: str = "epilogue") -> "FusedGather":
        """Switch this shard to the fused gather (see FusedGather; mode "epilogue" or "blocks");
        returns it."""
        if self.engine is None:
            raise ValueError("the fused gather needs the shard's DoseEngine")
        self.fused = FusedGather(self.engine, self.bounds, self.device, group, mode=mode)
        return self.fused

    def close(self):
        if getattr(self, "fused", None) is not None:
            self.fused.close()
            self.fused = None
        if self.engine is not None:
            self.engine.close()


class FusedGather:
    """The d all-gather fused into the dose kernels over peer memory.

    Every rank allocates a full-d buffer (``PeerBuffer``), the 64-byte CUDA IPC handles are
    exchanged with ``all_gather_object`` (host plumbing, once), each rank maps its peers' buffers
    and registers all ``world`` buffers with ``dg_set_gather_targets``.  A dose then stores each
    finished row of this rank's shard into every rank's full d straight from the kernel epilogue
    (NVLink / NVSwitch P2P stores), so the exchange overlaps the SpMV instead of following it as
    a separate NCCL all-gather.  After ``dose`` returns on every rank (stream synchronised, then
    a barrier), ``full`` holds the complete d on this rank.

    ``mode="blocks"``: the same buffers, filled by the copy engines instead of the kernels'
    epilogues -- each row block of this rank's d is copied to every rank's full d as soon as the
    tile kernel publishes the block (``dg_set_block_targets``): coalesced DMA over NVLink,
    overlapped with the later blocks' tiles, no SM time and no scalar remote stores.
    """

    def __init__(self, engine: DoseEngine, bounds, device: int, group=None,
                 mode: str = "epilogue"):
        if mode not in ("epilogue", "blocks"):
            raise ValueError(f"unknown fused-gather mode {mode!r}")
        import torch.distributed as dist

        from .dose import PeerBuffer

        self.engine, self.group, self.device = engine, group, device
        n = int(bounds[-1])
        self.mine = PeerBuffer(n, device)
        handles = [None] * dist.get_world_size(group)
        dist.all_gather_object(handles, self.mine.handle, group=group)
        me = dist.get_rank(group)
        self.peers = [None if g == me else PeerBuffer.open(h, n, device)
                      for g, h in enumerate(handles)]
        ptrs = [self.mine.ptr if g == me else self.peers[g].ptr for g in range(len(handles))]
        self.mode = mode
        if mode == "blocks":
            engine.set_block_targets(ptrs)
        else:
            engine.set_gather_targets(ptrs)
        self.full = self.mine.tensor()

    @staticmethod
    def preflight(device: int, group=None) -> bool:
        """Whether every rank can export and map CUDA IPC buffers (the same answer on every rank:
        a failure on one rank must not leave the others blocked in a collective).  Allocates,
        exchanges and maps a one-element buffer per rank."""
        import torch
        import torch.distributed as dist

        from .dose import PeerBuffer

        mine, handle = None, None
        try:
            mine = PeerBuffer(1, device)
            handle = mine.handle
        except Exception:
            handle = None
        handles = [None] * dist.get_world_size(group)
        dist.all_gather_object(handles, handle, group=group)
        me = dist.get_rank(group)
        ok, opened = all(h is not None for h in handles), []
        if ok:
            try:
                opened = [PeerBuffer.open(h, 1, device) for g, h in enumerate(handles) if g != me]
            except Exception:
                ok = False
        flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=f"cuda:{device}")
        if dist.get_backend(group) == "gloo":
            flag = flag.cpu()
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
        for p in opened:
            p.close()
        dist.barrier(group=group)
        if mine is not None:
            mine.close()
        return bool(flag.item())

    def dose(self, x, y_local, *, stream: int = 0):
        """This rank's slice into y_local and into every rank's full d; returns this rank's full
        d once every rank has finished (stream sync + barrier).  The returned tensor is read-only
        (its empty rows are zero-filled once, at the first dose, and never rewritten) and valid
        until the next ``dose`` call: that call first waits at a barrier for every rank (so no
        rank is still reading its full d from the previous dose when the peers' kernels start
        overwriting it), then overwrites it."""
        import torch
        import torch.distributed as dist

        own = not stream
        if own:
            stream = _torch_stream(self.device)
        # write-after-read: every rank is done with the previous full d before anyone writes it
        dist.barrier(group=self.group)
        self.engine.dose_device(x.data_ptr(), x.numel(), y_local.data_ptr(), stream=stream,
                                sync=False)
        if own:
            torch.cuda.current_stream(self.device).synchronize()
        else:
            torch.cuda.ExternalStream(stream).synchronize()
        dist.barrier(group=self.group)
        return self.full

    def close(self):
        import torch.distributed as dist

        if self.engine is not None and self.engine._h:
            if self.mode == "blocks":
                self.engine.set_block_targets([])
            else:
                self.engine.set_gather_targets([])
        # peers must stop writing into our buffer before it is freed
        if dist.is_initialized():
            dist.barrier(group=self.group)
        for p in self.peers:
            if p is not None:
                p.close()
        self.peers = []
        if dist.is_initialized():
            dist.barrier(group=self.group)
        self.full = None
        self.mine.close()
