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


VCR_HALO = 2  # z planes each rank receives from each neighbour (gpair_vcr.cu)


def slab_shard(grid, world: int, rank: int) -> tuple[int, int]:
    """Whole-z-plane split of the voxel grid (nx, ny, nz) for kernel sharding
    with lam > 0 (row f2): rank g owns the planes [z0, z0 + nz_g), ranks in z
    order, every rank >= VCR_HALO planes (the halo gpair_iterate exchanges).
    Returns (z0, nz_g); its kernels are [z0 nx ny, (z0 + nz_g) nx ny)."""
    nz = int(grid[2])
    if world < 1 or not (0 <= rank < world) or nz < VCR_HALO * world:
        raise ValueError(f"cannot split {nz} z planes over {world} ranks with >= {VCR_HALO} each")
    z0, z1 = rank * nz // world, (rank + 1) * nz // world
    return z0, z1 - z0


def halo_plan(world: int, rank: int, nz_own: int):
    """The z-slab halo exchange of gpair_iterate (gpair_api.cu vcr_sharded) as
    (peer, send planes [a, b) of the own slab, receive offset in planes of the
    extended buffer) triples; the extended buffer is [lower halo | own | upper
    halo] with lower = VCR_HALO planes if rank > 0 and upper likewise if
    rank < world - 1."""
    lo = VCR_HALO if rank > 0 else 0
    plan = []
    if rank > 0:
        plan.append((rank - 1, (0, VCR_HALO), 0))
    if rank < world - 1:
        plan.append((rank + 1, (nz_own - VCR_HALO, nz_own), lo + nz_own))
    return lo, plan


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
