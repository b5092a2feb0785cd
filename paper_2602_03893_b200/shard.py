"""Host-side multi-GPU plumbing: kernel sharding and the NCCL
communicator bootstrap for libgpair.  No arithmetic of the method lives here.

Kernel sharding: rank g owns the contiguous kernel range [lo, hi) of the
caller's order (z-slabs of the paper's voxel grid, i = ix + nx (iy + ny iz)).
The forward is linear in the kernels, so partial signals add; the one
collective is the all-reduce of y inside gpair_forward / gpair_iterate.
"""
from __future__ import annotations


def kernel_shard(M: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous split of M kernels over `world` ranks."""
    if world < 1 or not (0 <= rank < world) or M < world:
        raise ValueError(f"cannot shard {M} kernels over {world} ranks (rank {rank})")
    return rank * M // world, (rank + 1) * M // world


def nccl_bootstrap(dist, rank: int, world: int, unique_id_fn, comm_init_fn):
    """Rank 0 creates the 128-byte ncclUniqueId; torch.distributed broadcasts
    it; every rank initialises a library-owned communicator.  `dist` is
    torch.distributed (any backend), the two callables are gpair.nccl_unique_id
    and gpair.nccl_comm_init (injectable for CPU tests)."""
    obj = [unique_id_fn() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    uid = obj[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != 128:
        raise RuntimeError("bad ncclUniqueId broadcast")
    return comm_init_fn(world, bytes(uid), rank)


def max_over_ranks(dist, value: float, device=None) -> float:
    """Max of a per-rank scalar (timings are reported as the max over ranks)."""
    import torch

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
