"""The kernel-sharded (collective) path of the library on one GPU.

gpair_forward / gpair_iterate at world > 1 all-reduce y with NCCL in place,
compute the residual in a separate kernel (k_residual) on every rank, and (lam
> 0) exchange R_VCR halos and all-reduce its value (superposition
P:242).  NCCL refuses two ranks on one device, so on this
one-GPU harness the same code runs with GPAIR_COLLECTIVE and a 1-rank NCCL
communicator, whose collectives are identities: every branch of the world > 1
path executes (all-reduce of y, k_residual, the pipelined per-group
all-reduces, gpair_vcr_prepare's agreement all-reduce, the 8-byte R_VCR
all-reduce) and must reproduce the world = 1 path bit for bit where the
arithmetic is the same, and the oracle within the common gate.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from oracle import ir, vcr  # noqa: E402
from paper_2602_03893_b200 import gpair, inputs  # noqa: E402
from tests_common import T, assert_parity  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_03893_b200 import build

    build.build()


@pytest.fixture(scope="module")
def comm():
    c = gpair.nccl_comm_init(1, gpair.nccl_unique_id(), 0)
    yield c
    gpair.nccl_comm_destroy(c)


def case():
    """TAB / LCF-eligible, oracle-cheap: 16^3 kernels, 64-sensor hemisphere, W = 16."""
    c = inputs.grid_centers(16, 16, 16, 1e-4)
    s = inputs.hemisphere(64, 60e-3)
    op = dict(sigma=1e-4, v=1500.0, fs=40e6, n_samples=2048, t0=0.0, k=3.0)
    return c, s, op


def ctx_of(c, s, op, comm=None, monkeypatch=None, pipeline=False):
    if monkeypatch is not None:
        monkeypatch.setenv("GPAIR_PIPELINE", "1" if pipeline else "0")
    kw = dict(sigma=op["sigma"], v=op["v"], fs=op["fs"], n_samples=op["n_samples"], t0=op["t0"], k=op["k"])
    if comm is not None:
        kw.update(nccl_comm=comm, flags=gpair.COLLECTIVE)
    return gpair.Context(T(c), T(s), **kw)


def test_collective_flag_needs_a_matching_communicator(comm):
    c, s, op = case()
    with pytest.raises(gpair.GpairError) as e:  # GPAIR_COLLECTIVE without a communicator
        gpair.Context(T(c), T(s), sigma=op["sigma"], v=op["v"], fs=op["fs"], n_samples=op["n_samples"],
                      flags=gpair.COLLECTIVE)
    assert e.value.status == gpair.ERR_INVALID_ARGUMENT
    with pytest.raises(gpair.GpairError) as e:  # communicator of 1 rank, world = 2
        gpair.Context(T(c), T(s), sigma=op["sigma"], v=op["v"], fs=op["fs"], n_samples=op["n_samples"],
                      rank=0, world=2, nccl_comm=comm)
    assert e.value.status == gpair.ERR_INVALID_ARGUMENT
    ctx = ctx_of(c, s, op, comm)
    assert ctx.info()["collective"] == 1
    ctx.close()
    ctx = ctx_of(c, s, op)
    assert ctx.info()["collective"] == 0
    ctx.close()


def test_forward_adjoint_collective_equals_world1(comm):
    c, s, op = case()
    x = T(inputs.dense_amplitudes(c.shape[1]))
    d = T(inputs.residual(s.shape[1], op["n_samples"]))
    a, b = ctx_of(c, s, op), ctx_of(c, s, op, comm)
    ya, yb = a.forward(x), b.forward(x)
    torch.cuda.synchronize()
    assert torch.equal(ya, yb)
    assert torch.equal(a.adjoint(d), b.adjoint(d))
    assert_parity(yb.cpu().numpy(), oracle.forward(c, x.cpu().numpy(), s, **op), "collective forward")
    a.close()
    b.close()


def _iterate(ctx, c, s, op, mode, lam=0.0, grid=None, steps=2):
    M = c.shape[1]
    rng = np.random.default_rng(17)
    b = oracle.forward(c, inputs.vessel_phantom(16, 16, 16) + 0.1 * rng.random(M).astype(np.float32), s,
                       **op).astype(np.float32)
    z0 = rng.uniform(0.2, 0.9, M).astype(np.float32)
    z, m, v = T(z0), torch.zeros(M, device="cuda"), torch.zeros(M, device="cuda")
    y = torch.zeros(s.shape[1] * op["n_samples"], device="cuda")
    loss = torch.zeros(1, device="cuda")
    kw = dict(lam=lam, beta=0.5, eps_reg=1e-8, grid=grid, z0=0) if lam > 0 else {}
    losses = []
    for t in range(steps):
        ctx.iterate(z, m, v, T(b), lr=0.01, step=t + 1, mode=mode, loss_out=loss, signals_out=y, **kw)
        losses.append(loss.item())
    torch.cuda.synchronize()
    return dict(z=z.cpu().numpy(), m=m.cpu().numpy(), v=v.cpu().numpy(), y=y.cpu().numpy(), loss=np.array(losses),
                b=b, z0=z0)


@pytest.mark.parametrize("pipeline", [False, True])
@pytest.mark.parametrize("mode", [0, 1])
def test_iterate_collective_equals_world1(comm, monkeypatch, pipeline, mode):
    """Two iterations through the collective branch (NCCL all-reduce of y, k_residual,
    and with the pipeline the per-sensor-group all-reduces on the internal stream)
    reproduce the world = 1 path: state and y bit for bit, loss to fp64 summation order."""
    c, s, op = case()
    ra = _iterate(ctx_of(c, s, op, monkeypatch=monkeypatch, pipeline=pipeline), c, s, op, mode)
    rb = _iterate(ctx_of(c, s, op, comm, monkeypatch=monkeypatch, pipeline=pipeline), c, s, op, mode)
    for key in ("z", "m", "v", "y"):
        assert np.array_equal(ra[key], rb[key]), key
    np.testing.assert_allclose(rb["loss"], ra["loss"], rtol=1e-6)
    # and the first iteration against the oracle (x = z0 before the update)
    geom = {"centers": c, "sensors": s, "op": op}
    hp = ir.Hyper(mode="npc" if mode == 0 else "clamp")
    L_ref, _, _ = ir.loss_and_grad(rb["z0"].astype(np.float64), rb["b"].astype(np.float64), geom, hp)
    assert abs(rb["loss"][0] - L_ref) / L_ref <= 1e-5


@pytest.mark.parametrize("mode", [0, 1])
def test_iterate_vcr_collective(comm, mode):
    """lam > 0 on the collective path: gpair_vcr_prepare's agreement all-reduce, the slab
    kernels over the whole grid, and the 8-byte fp64 all-reduce of R_VCR; the state
    equals the world = 1 path bit for bit and the loss includes lam R_VCR (oracle)."""
    c, s, op = case()
    grid = (16, 16, 16)
    lam = 3e-6
    a = ctx_of(c, s, op)
    b = ctx_of(c, s, op, comm)
    with pytest.raises(gpair.GpairError) as e:  # the collective path needs the prepared layout
        _iterate(b, c, s, op, mode, lam=lam, grid=grid, steps=1)
    assert e.value.status == gpair.ERR_INVALID_ARGUMENT
    with pytest.raises(gpair.GpairError):
        b.vcr_prepare((16, 16, 15))
    b.vcr_prepare(grid, 0)
    a.vcr_prepare(grid, 0)  # optional at world 1 (pre-allocation only)
    ra = _iterate(a, c, s, op, mode, lam=lam, grid=grid)
    rb = _iterate(b, c, s, op, mode, lam=lam, grid=grid)
    for key in ("z", "m", "v", "y"):
        assert np.array_equal(ra[key], rb[key]), key
    np.testing.assert_allclose(rb["loss"], ra["loss"], rtol=1e-6)
    x0 = ir.npc(rb["z0"].astype(np.float64)) if mode == 0 else rb["z0"].astype(np.float64)
    y0 = oracle.forward(c, x0, s, **op)
    R0, _ = vcr.r_vcr(x0, grid, 0.5, 1e-8)
    L_ref = float(np.mean((y0 - rb["b"]) ** 2)) + lam * R0
    assert abs(rb["loss"][0] - L_ref) / L_ref <= 1e-5
    a.close()
    b.close()
