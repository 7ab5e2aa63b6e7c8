"""Multi-GPU plumbing for the batched search: one process per
GPU, the index replicated on every rank, the query batch split into
contiguous ranges; no collective on the data path.  torch.distributed is used
only for barriers and the max-over-ranks timing reduction (NCCL on GPUs, gloo
in the CPU tests)."""
from __future__ import annotations

import os


def shard_range(count: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [lo, hi) of `count` queries owned by `rank` (ceil split)."""
    per = (count + world - 1) // world
    lo = min(count, rank * per)
    return lo, min(count, lo + per)


def env_world() -> tuple[int, int, int]:
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


class Group:
    """Barrier / max / broadcast over the process group (no-ops when world == 1)."""

    def __init__(self, world: int, device: str = "cpu"):
        self.world = world
        self.device = device

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier()

    def _reduce(self, x: float, op) -> float:
        if self.world == 1:
            return float(x)
        import torch
        import torch.distributed as dist
        t = torch.tensor([float(x)], dtype=torch.float64, device=self.device)
        dist.all_reduce(t, op=op)
        return float(t.item())

    def max(self, x: float) -> float:
        import torch.distributed as dist
        return self._reduce(x, dist.ReduceOp.MAX if self.world > 1 else None)

    def sum(self, x: float) -> float:
        import torch.distributed as dist
        return self._reduce(x, dist.ReduceOp.SUM if self.world > 1 else None)

    def bcast(self, x: float, src: int = 0) -> float:
        if self.world == 1:
            return float(x)
        import torch
        import torch.distributed as dist
        t = torch.tensor([float(x)], dtype=torch.float64, device=self.device)
        dist.broadcast(t, src)
        return float(t.item())


def build_comm(world: int, rank: int, device: int):
    """The library's NCCL communicator for a sharded build (fg_comm_init):
    rank 0 draws the unique id, torch.distributed broadcasts it (any backend)."""
    from .fusegraph import Comm
    if world == 1:
        return None
    import torch.distributed as dist
    box = [Comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0)
    return Comm(world, rank, box[0], device)


def vertex_ranges(n: int, world: int) -> list[tuple[int, int]]:
    """Node ranges of the sharded build: rank r owns [r*cn, min(n, (r+1)*cn)),
    cn = ceil(n / world) (fg_index_build_sharded, include/fg_b200.h)."""
    cn = (n + world - 1) // world
    return [(min(n, r * cn), min(n, (r + 1) * cn)) for r in range(world)]
