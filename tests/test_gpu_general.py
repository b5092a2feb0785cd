"""GPU parity of the general operator: per-kernel sigma_i
(reading N2) and the near-field operator, Eq. 6 with both terms (PAPER.md
P:264-276, readings N1-N3), through the C ABI against the fp64 oracle
(`oracle.forward/adjoint(..., sigmas=, near_field=)`, pinned in
tests/test_oracle_nearfield.py).  Same gates as the direct operator:
rel L2 <= 1e-5, elementwise <= 1e-4 above 1e-3 of peak on every output (tests_common).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from oracle import ir  # noqa: E402
from paper_2602_03893_b200 import gpair, inputs  # noqa: E402

from tests_common import T, assert_parity, assert_state_update, dev  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_03893_b200 import build

    build.build()


def _ctx(c, s, op, sigmas=None, near_field=False):
    return gpair.Context(T(c), T(s), sigma=op["sigma"], v=op["v"], fs=op["fs"], n_samples=op["n_samples"],
                         t0=op["t0"], k=op["k"], sigmas=None if sigmas is None else T(sigmas.astype(np.float32)),
                         near_field=near_field)


def _kw(op):
    return {k: v for k, v in op.items() if k != "n_samples"}


def _check(c, s, op, sigmas=None, near_field=False, seed=0, what=""):
    ctx = _ctx(c, s, op, sigmas, near_field)
    M = c.shape[1]
    x = np.random.default_rng(seed).random(M).astype(np.float32)
    sg = None if sigmas is None else sigmas.astype(np.float32).astype(np.float64)
    y = ctx.forward(T(x)).cpu().numpy()
    y_ref = oracle.forward(c, x, s, sigmas=sg, near_field=near_field, **op)
    assert_parity(y, y_ref, f"{what} forward")
    d = inputs.residual(s.shape[1], op["n_samples"], seed=seed + 1)
    g = ctx.adjoint(T(d)).cpu().numpy()
    g_ref = oracle.adjoint(c, d, s, sigmas=sg, near_field=near_field, **_kw(op))
    assert_parity(g, g_ref, f"{what} adjoint")
    return ctx


def _sigmas(M, base, seed, lo=0.7, hi=1.3):
    return (np.random.default_rng(seed).uniform(lo, hi, M) * base).astype(np.float32)


def test_per_kernel_sigma_cfg1():
    cfg = inputs.CONFIGS["cfg1"]
    c, s, op = cfg.centers(), cfg.sensors(), cfg.op_kwargs()
    ctx = _check(c, s, op, sigmas=_sigmas(cfg.M, op["sigma"], 1), what="cfg1 sigma_i")
    assert ctx.info()["general"] == 1 and ctx.info()["near_pairs"] == 0
    with pytest.raises(gpair.GpairError):
        ctx.count_pair_samples()


@pytest.mark.parametrize("seed", range(6))
def test_per_kernel_sigma_random_suite(seed):
    """Ragged grids, jitter, t0 > 0, record clipping at both ends."""
    c, s, op = inputs.random_suite_case(seed)
    # keep every pair far: sigma_i <= sigma (the suite's geometry is valid for sigma)
    _check(c, s, op, sigmas=_sigmas(c.shape[1], op["sigma"], seed, 0.5, 1.0), seed=seed, what=f"suite {seed} sigma_i")


def _near_case(seed, n_inside=8, t0=0.0, grid=(12, 12, 12)):
    """A kernel grid with a far hemisphere plus sensors inside the volume."""
    rng = np.random.default_rng(100 + seed)
    c = inputs.grid_centers(*grid, 1e-4, jitter=0.2, seed=seed)
    far = inputs.hemisphere(40, 8e-3)
    half = 0.5 * 1e-4 * (np.array(grid) - 1)
    inside = (rng.uniform(-1, 1, (3, n_inside)) * half[:, None]).astype(np.float32)
    s = np.ascontiguousarray(np.concatenate([far, inside], axis=1))
    op = dict(sigma=1e-4, v=1500.0, fs=40e6, n_samples=256, t0=t0, k=3.0)
    return c, s, op


@pytest.mark.parametrize("seed", range(3))
def test_near_field(seed):
    c, s, op = _near_case(seed)
    ctx = _check(c, s, op, near_field=True, seed=seed, what=f"near field {seed}")
    info = ctx.info()
    assert info["near_pairs"] > 0 and info["near_rows"] == 8


def test_near_field_with_sigmas_and_negative_t0():
    c, s, op = _near_case(7, t0=-2e-7)
    _check(c, s, op, sigmas=_sigmas(c.shape[1], op["sigma"], 7), near_field=True, seed=7, what="near sigma_i t0<0")


def test_near_field_without_near_pairs_matches_exact_operator():
    cfg = inputs.CONFIGS["cfg1"]
    c, s, op = cfg.centers(), cfg.sensors(), cfg.op_kwargs()
    ctx = _check(c, s, op, near_field=True, what="cfg1 near-field flag")
    assert ctx.info()["near_pairs"] == 0


def test_near_field_rejects_r_zero():
    c, s, op = _near_case(0, n_inside=0)
    s = np.ascontiguousarray(np.concatenate([s, c[:, 5:6]], axis=1))  # a sensor exactly on a kernel centre
    with pytest.raises(gpair.GpairError) as e:
        _ctx(c, s, op, near_field=True)
    assert e.value.status == gpair.ERR_GEOMETRY
    # without the flag the far-field check rejects it as before
    with pytest.raises(gpair.GpairError):
        _ctx(c, s, op)


@pytest.mark.parametrize("mode", [0, 1])
def test_iterate_general_teacher_forced(mode):
    """One Alg. 2 iteration on the near-field + sigma_i operator."""
    c, s, op = _near_case(3, n_inside=4)
    sig = _sigmas(c.shape[1], op["sigma"], 3)
    sg = sig.astype(np.float64)
    ctx = _ctx(c, s, op, sig, near_field=True)
    rng = np.random.default_rng(5)
    M = c.shape[1]
    x_true = rng.random(M)
    b = oracle.forward(c, x_true, s, sigmas=sg, near_field=True, **op).astype(np.float32)
    z0 = rng.uniform(0.2, 0.9, M).astype(np.float32)
    hp = ir.Hyper(mode="npc" if mode == 0 else "clamp")
    x0 = ir.npc(z0.astype(np.float64)) if mode == 0 else z0.astype(np.float64)
    y_ref = oracle.forward(c, x0, s, sigmas=sg, near_field=True, **op)
    r = y_ref - b
    N = r.size
    L_ref = float(np.sum(r * r) / N)
    gx = oracle.adjoint(c, (2.0 / N) * r, s, sigmas=sg, near_field=True, **_kw(op))
    gz = ir.npc_chain(gx, z0.astype(np.float64), hp.eps_npc) if mode == 0 else gx
    m0 = (0.5 * gz).astype(np.float32)
    v0 = (gz * gz).astype(np.float32)
    lr = 0.1 if mode == 0 else float(0.05 * np.abs(z0).max() / np.abs(gz).max())  # step >> ulp(z)
    zt, mt, vt = T(z0), T(m0), T(v0)
    loss = torch.empty(1, device=dev())
    yo = torch.empty((s.shape[1], op["n_samples"]), device=dev())
    ctx.iterate(zt, mt, vt, T(b), lr=lr, step=3, mode=mode, signals_out=yo, loss_out=loss)
    torch.cuda.synchronize()
    assert_parity(yo.cpu().numpy(), y_ref, "general iterate signals")
    assert abs(loss.item() - L_ref) <= 1e-5 * L_ref
    if mode == 0:
        z_ref, _, _ = ir.adam_update(z0.astype(np.float64), m0.astype(np.float64), v0.astype(np.float64), gz, lr, 3, hp)
    else:
        z_ref = np.maximum(z0 - lr * gz, 0.0)
    assert_state_update(zt.cpu().numpy(), z0, z_ref, "general iterate step")
