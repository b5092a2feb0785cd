"""world_size-2 gloo tests of the N > 1 host path on CPU (no GPU needed):
kernel sharding, the ncclUniqueId broadcast bootstrap, max-over-ranks timing,
and that per-shard forwards summed by an all-reduce equal the full forward
(the algebra the kernel-sharded GPU path relies on; oracle as the operator)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_03893_b200 import inputs
from paper_2602_03893_b200.shard import VCR_HALO, halo_plan, kernel_shard, max_over_ranks, nccl_bootstrap, slab_shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle

        oracle.set_threads(1)
        cfg = inputs.CONFIGS["cfg1"]
        c, s, op = cfg.centers(), cfg.sensors(), cfg.op_kwargs()
        x = inputs.dense_amplitudes(cfg.M)
        lo, hi = kernel_shard(cfg.M, world, rank)
        y = oracle.forward(np.ascontiguousarray(c[:, lo:hi]), x[lo:hi], s, **op)
        t = torch.from_numpy(y)
        dist.all_reduce(t)  # the one collective of the sharded path
        calls = []

        def uid():
            calls.append("uid")
            return bytes(range(128))

        def init(w, u, r):
            calls.append(("init", w, r))
            return (w, u, r)

        comm = nccl_bootstrap(dist, rank, world, uid, init)
        m = max_over_ranks(dist, 1.0 + rank)
        q.put((rank, t.numpy(), comm, calls, m, (lo, hi)))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharded_forward_and_bootstrap():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda r: r[0])
    import oracle

    cfg = inputs.CONFIGS["cfg1"]
    y_full = oracle.forward(cfg.centers(), inputs.dense_amplitudes(cfg.M), cfg.sensors(), **cfg.op_kwargs())
    for rank, y, comm, calls, m, rng in res:
        assert np.linalg.norm(y - y_full) <= 1e-12 * np.linalg.norm(y_full)
        assert comm == (world, bytes(range(128)), rank)
        assert calls[-1] == ("init", world, rank)
        assert ("uid" in calls) == (rank == 0)
        assert m == 2.0
    assert res[0][5] == (0, cfg.M // 2) and res[1][5] == (cfg.M // 2, cfg.M)


def test_kernel_shard_covers_exactly_once():
    for M in (512, 1000, 8388608):
        for world in (1, 2, 3, 8):
            spans = [kernel_shard(M, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == M
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [h - l for l, h in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        kernel_shard(4, 8, 0)


def _vcr_worker(rank, world, port, q):
    """One rank of the kernel-sharded R_VCR gradient (row f2): exchange the
    z-slab halos with gloo send/recv following shard.halo_plan (the protocol
    gpair_iterate runs over NCCL), then evaluate the own planes from the
    extended buffer alone: every plane outside it is replaced by noise before
    the (whole-grid) oracle runs, so a missing or misplaced halo plane shows."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import vcr

        dims = (5, 4, 13)
        nx, ny, nz = dims
        P = nx * ny
        full = np.random.default_rng(7).uniform(0.0, 1.0, (nz, ny, nx))
        z0, nzo = slab_shard(dims, world, rank)
        own = torch.from_numpy(np.ascontiguousarray(full[z0:z0 + nzo]))  # this rank's state only
        lo, plan = halo_plan(world, rank, nzo)
        hi = VCR_HALO if rank < world - 1 else 0
        ext = torch.zeros((lo + nzo + hi, ny, nx), dtype=torch.float64)
        ext[lo:lo + nzo] = own
        reqs = []
        for peer, (a, b), off in plan:
            reqs.append(dist.isend(own[a:b].contiguous(), peer))
        recv = []
        for peer, (a, b), off in plan:
            buf = torch.empty((VCR_HALO, ny, nx), dtype=torch.float64)
            reqs.append(dist.irecv(buf, peer))
            recv.append((off, buf))
        for r in reqs:
            r.wait()
        for off, buf in recv:
            ext[off:off + VCR_HALO] = buf
        img = np.random.default_rng(100 + rank).uniform(0.0, 1.0, (nz, ny, nx))  # noise outside the buffer
        img[z0 - lo:z0 + nzo + hi] = ext.numpy()
        _, g = vcr.r_vcr(img.ravel(), dims, 0.5, 1e-3)
        q.put((rank, z0, nzo, g[z0 * P:(z0 + nzo) * P]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_vcr_halo_exchange_protocol(world):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_vcr_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle import vcr

    dims = (5, 4, 13)
    full = np.random.default_rng(7).uniform(0.0, 1.0, (dims[2], dims[1], dims[0]))
    _, g_full = vcr.r_vcr(full.ravel(), dims, 0.5, 1e-3)
    assert [r[1] for r in res] == sorted(r[1] for r in res) and res[0][1] == 0
    assert sum(r[2] for r in res) == dims[2]
    g = np.concatenate([r[3] for r in res])
    assert np.array_equal(g, g_full)


def test_slab_shard_rules():
    assert [slab_shard((4, 4, 16), 8, r) for r in range(8)] == [(2 * r, 2) for r in range(8)]
    assert [slab_shard((4, 4, 13), 3, r) for r in range(3)] == [(0, 4), (4, 4), (8, 5)]
    with pytest.raises(ValueError):
        slab_shard((4, 4, 7), 4, 0)  # fewer than VCR_HALO planes per rank
    assert halo_plan(1, 0, 5) == (0, [])
    assert halo_plan(3, 1, 5) == (2, [(0, (0, 2), 0), (2, (3, 5), 7)])
