"""GPU parity of the VCR regulariser (row f2; Eqs. 20-23,
P:457-481) through the C ABI (gpair_vcr, gpair_iterate with lam > 0)
against oracle/vcr.py and oracle/ir.py (readings V1-V4 of DESIGN.md).

Inputs are fp32 images cast exactly to fp64 for the oracle.  Gate: the
north_star's rel L2 <= 1e-5 on the gradient, 1e-6 relative on the value (an
fp64-accumulated sum of positive fp32 terms), and the common elementwise
gate of tests_common on every gradient / state vector.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from oracle import ir, vcr  # noqa: E402
from paper_2602_03893_b200 import gpair, inputs  # noqa: E402

from tests_common import T, assert_parity, assert_state_update, dev  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_03893_b200 import build

    build.build()


@pytest.fixture(scope="module")
def ctx():
    cfg = inputs.CONFIGS["cfg1"]
    op = cfg.op_kwargs()
    return gpair.Context(T(cfg.centers()), T(cfg.sensors()), sigma=op["sigma"], v=op["v"], fs=op["fs"],
                         n_samples=op["n_samples"], t0=op["t0"], k=op["k"])


def _gpu_vcr(ctx, x, dims, beta, eps):
    M = int(np.prod(dims))
    g = torch.empty(M, device=dev())
    val = torch.empty(1, device=dev())
    ctx.vcr(T(x.astype(np.float32)), dims, beta=beta, eps=eps, grad=g, value=val)
    torch.cuda.synchronize()
    return float(val.item()), g.cpu().numpy()


DIMS = [(1, 1, 1), (2, 2, 2), (3, 1, 6), (5, 3, 2), (2, 7, 3), (16, 16, 16), (33, 17, 9), (70, 50, 40)]


@pytest.mark.parametrize("dims", DIMS)
@pytest.mark.parametrize("beta,eps", [(0.0, 1e-3), (0.5, 1e-3), (1.0, 1e-8)])
def test_vcr_random_image(ctx, dims, beta, eps):
    rng = np.random.default_rng(hash((dims, beta)) % 2**32)
    M = int(np.prod(dims))
    x = rng.uniform(0.0, 1.0, M).astype(np.float32)
    v_ref, g_ref = vcr.r_vcr(x.astype(np.float64), dims, beta, eps)
    v, g = _gpu_vcr(ctx, x, dims, beta, eps)
    assert abs(v - v_ref) <= 1e-6 * abs(v_ref), (v, v_ref)
    if M > 1:
        assert_parity(g, g_ref, f"VCR grad {dims}")
    else:
        assert np.abs(g).max() == 0.0


def test_vcr_vessel_phantom(ctx):
    """Structured input of the paper's kind (vessel tubes)."""
    dims = (40, 40, 20)
    x = inputs.vessel_phantom(*dims).astype(np.float32)
    v_ref, g_ref = vcr.r_vcr(x.astype(np.float64), dims, 0.3, 1e-3)
    v, g = _gpu_vcr(ctx, x, dims, 0.3, 1e-3)
    assert abs(v - v_ref) <= 1e-6 * abs(v_ref)
    assert_parity(g, g_ref, "VCR grad phantom")


def test_vcr_constant_image_closed_form(ctx):
    """R(const) = 2 M sqrt(eps) for beta = 1 and a zero gradient (pin of the
    oracle reproduced on the GPU)."""
    dims = (9, 8, 7)
    M = int(np.prod(dims))
    v, g = _gpu_vcr(ctx, np.full(M, 0.75, np.float32), dims, 1.0, 1e-4)
    assert abs(v - 2 * M * 1e-2) <= 1e-6 * 2 * M * 1e-2
    assert np.abs(g).max() == 0.0


SLABS = [((6, 5, 14), [0, 4, 6, 9, 14]), ((6, 5, 14), [0, 1, 2, 3, 11, 12, 13, 14]), ((33, 17, 9), [0, 2, 5, 9]),
         ((70, 50, 40), [0, 5, 10, 15, 20, 25, 30, 35, 40]), ((4, 3, 2), [0, 1, 2]), ((3, 4, 5), [0, 5])]


@pytest.mark.parametrize("dims,cuts", SLABS)
@pytest.mark.parametrize("halo", ["exact", "whole"])
def test_vcr_slabs_match_whole_grid(ctx, dims, cuts, halo):
    """Kernel-sharded R_VCR (row f2, gpair_vcr_slab): each z slab, given its
    2-plane halo ('exact') or the whole grid ('whole'), yields the own-plane
    entries of the whole-grid gradient, and the slab values add up to the
    whole-grid value (oracle/vcr.py on the whole grid)."""
    nx, ny, nz = dims
    P = nx * ny
    rng = np.random.default_rng(len(cuts) + nz)
    x = rng.uniform(0.0, 1.0, P * nz).astype(np.float32)
    v_ref, g_ref = vcr.r_vcr(x.astype(np.float64), dims, 0.6, 1e-3)
    xs = T(x)
    total, grads = 0.0, []
    for z0, z1 in zip(cuts[:-1], cuts[1:]):
        e0, e1 = (max(0, z0 - 2), min(nz, z1 + 2)) if halo == "exact" else (0, nz)
        g = torch.empty(P * (z1 - z0), device=dev())
        val = torch.empty(1, device=dev())
        ctx.vcr_slab(xs[e0 * P:e1 * P].contiguous(), dims, z0, z1 - z0, e0, beta=0.6, eps=1e-3, grad=g, value=val)
        torch.cuda.synchronize()
        total += float(val.item())
        grads.append(g.cpu().numpy())
    assert abs(total - v_ref) <= 1e-6 * abs(v_ref), (total, v_ref)
    assert_parity(np.concatenate(grads), g_ref, f"VCR slab grad {dims} {cuts}")


def test_vcr_whole_slab_is_bit_identical_to_gpair_vcr(ctx):
    """The whole grid as one slab runs the same arithmetic as gpair_vcr."""
    dims = (33, 17, 9)
    M = int(np.prod(dims))
    x = T(np.random.default_rng(5).uniform(0.0, 1.0, M).astype(np.float32))
    g1, g2 = torch.empty(M, device=dev()), torch.empty(M, device=dev())
    v1, v2 = torch.empty(1, device=dev()), torch.empty(1, device=dev())
    ctx.vcr(x, dims, beta=0.4, eps=1e-4, grad=g1, value=v1)
    ctx.vcr_slab(x, dims, 0, dims[2], 0, beta=0.4, eps=1e-4, grad=g2, value=v2)
    torch.cuda.synchronize()
    assert torch.equal(g1, g2) and torch.equal(v1, v2)


def test_vcr_slab_invalid_arguments(ctx):
    dims = (4, 4, 10)
    x = torch.zeros(16 * 10, device=dev())
    g = torch.empty(16 * 3, device=dev())
    with pytest.raises(gpair.GpairError):  # halo not covered (needs planes 2..9 for the slab 4..7)
        ctx.vcr_slab(x[16 * 3:16 * 9].contiguous(), dims, 4, 3, 3, beta=1.0, grad=g)
    with pytest.raises(gpair.GpairError):  # slab outside the grid
        ctx.vcr_slab(x, dims, 8, 3, 0, beta=1.0, grad=g)
    ctx.vcr_slab(x[16 * 2:16 * 9].contiguous(), dims, 4, 3, 2, beta=1.0, grad=g)


def test_vcr_invalid_arguments(ctx):
    x = torch.zeros(8, device=dev())
    with pytest.raises(gpair.GpairError):
        ctx.vcr(x, (2, 2, 2), beta=1.0, eps=0.0, value=torch.empty(1, device=dev()))
    with pytest.raises(gpair.GpairError):
        ctx.vcr(x, (2, 0, 2), beta=1.0, eps=1e-8, value=torch.empty(1, device=dev()))


@pytest.mark.parametrize("mode", [0, 1])
def test_iterate_with_vcr_teacher_forced(mode):
    """One Alg. 2 iteration with lambda > 0 (Eq. 23): loss = data + lam R,
    gradient = A^T(2/N r) + lam grad R, then NPC chain + Adam / clamp."""
    cfg = inputs.CONFIGS["cfg1"]
    c, s, op = cfg.centers(), cfg.sensors(), cfg.op_kwargs()
    ctx = gpair.Context(T(c), T(s), sigma=op["sigma"], v=op["v"], fs=op["fs"], n_samples=op["n_samples"],
                        t0=op["t0"], k=op["k"])
    rng = np.random.default_rng(21)
    x_true = inputs.vessel_phantom(*cfg.grid) + 0.1 * rng.random(cfg.M).astype(np.float32)
    b = oracle.forward(c, x_true, s, **op).astype(np.float32)
    z0 = rng.uniform(0.2, 0.9, cfg.M).astype(np.float32)
    geom = {"centers": c, "sensors": s, "op": op}
    hp0 = ir.Hyper(mode="npc" if mode == 0 else "clamp")
    L0, _, _ = ir.loss_and_grad(z0.astype(np.float64), b.astype(np.float64), geom, hp0)
    # lambda so that lam R_VCR is comparable with the data term
    rv = vcr.r_vcr(ir.npc(z0.astype(np.float64)) if mode == 0 else z0.astype(np.float64), cfg.grid, 0.5, 1e-4)[0]
    lam = float(np.float32(L0 / rv))
    hp = ir.Hyper(mode=hp0.mode, lam=lam, beta=0.5, eps_reg=1e-4, dims=cfg.grid)
    _, gz0, _ = ir.loss_and_grad(z0.astype(np.float64), b.astype(np.float64), geom, hp)
    m0 = (0.5 * gz0 * rng.uniform(0.5, 1.5, cfg.M)).astype(np.float32)
    v0 = (gz0 * gz0 * rng.uniform(0.5, 1.5, cfg.M)).astype(np.float32)
    t_step = 4
    lr = gpair.cawr_lr(t_step - 1, 1e-4, 0.1, 50, 1)
    if mode == 1:  # projected step: take lr so that lr |g| is a visible fraction of z (fp32 z - lr g)
        lr = float(0.05 * np.abs(z0).max() / np.abs(gz0).max())
    zt, mt, vt = T(z0), T(m0), T(v0)
    loss = torch.empty(1, device=dev())
    ctx.iterate(zt, mt, vt, T(b), lr=lr, step=t_step, mode=mode, lam=lam, beta=0.5, eps_reg=1e-4, grid=cfg.grid,
                loss_out=loss)
    torch.cuda.synchronize()
    L_ref, gz_ref, _ = ir.loss_and_grad(z0.astype(np.float64), b.astype(np.float64), geom, hp)
    assert abs(loss.item() - L_ref) / L_ref <= 1e-5
    if mode == 0:
        z_ref, m_ref, _ = ir.adam_update(z0.astype(np.float64), m0.astype(np.float64), v0.astype(np.float64),
                                         gz_ref, lr, t_step, hp)
        assert_parity(mt.cpu().numpy() - 0.9 * m0, m_ref - 0.9 * m0, "Adam m increment")
        assert_state_update(zt.cpu().numpy(), z0, z_ref, "Adam z step")
    else:
        x_ref = np.maximum(z0 - lr * gz_ref, 0.0)
        assert_state_update(zt.cpu().numpy(), z0, x_ref, "clamp step")


def test_iterate_vcr_rejects_bad_grid(ctx):
    cfg = inputs.CONFIGS["cfg1"]
    z = torch.zeros(cfg.M, device=dev())
    b = torch.zeros((cfg.n_sensors, cfg.n_samples), device=dev())
    with pytest.raises(gpair.GpairError):
        ctx.iterate(z, z.clone(), z.clone(), b, lr=0.01, step=1, lam=1e-3, beta=0.5, eps_reg=1e-4,
                    grid=(cfg.grid[0], cfg.grid[1], cfg.grid[2] + 1))
