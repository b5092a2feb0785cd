"""GPU parity of the ASSA operator (Eqs. 8-17,
Algorithm 1) against the fp64 ASSA oracle, with the gates of the direct
operator (tests_common: rel L2 <= 1e-5 and elementwise <= 1e-4 on every
output); measured values are printed."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from oracle import ir  # noqa: E402
from paper_2602_03893_b200 import gpair, inputs  # noqa: E402
from tests_common import T, assert_parity, dev, sample_cols, sample_rows  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_03893_b200 import build

    build.build()


ADJ = {"mp": ({}, 4), "lane": ({"GPAIR_ADJ_NO_MP": "1"}, 0)}  # adjoint kernel: k_adjoint_mp / k_assa_adjoint


def make_ctx(c, s, op, nmin=25, monkeypatch=None, adj="mp"):
    if monkeypatch is not None:
        monkeypatch.delenv("GPAIR_ADJ_NO_MP", raising=False)
        for key, val in ADJ[adj][0].items():
            monkeypatch.setenv(key, val)
    return gpair.Context(T(c), T(s), sigma=op["sigma"], v=op["v"], fs=op["fs"], n_samples=op["n_samples"],
                         t0=op["t0"], k=op["k"], assa=True, assa_nmin=nmin)


def assa_kw(op, nmin=25):
    p = oracle.assa_params(op["sigma"], op["v"], op["fs"], op["k"], nmin)
    return p, dict(sigma=op["sigma"], v=op["v"], fs=op["fs"], t0=op["t0"], k=op["k"], alpha=p["alpha"], K=p["K"])


def impulse_count(c, s, op, alpha):
    c64, s64 = c.astype(np.float64), s.astype(np.float64)
    fs_up = alpha * op["fs"]
    n = 0
    for j in range(s.shape[1]):
        d = c64 - s64[:, j:j + 1]
        r = np.sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2])
        kk = np.floor((r / op["v"] - op["t0"]) * fs_up + 0.5)
        n += int(np.count_nonzero((kk >= 0) & (kk < alpha * op["n_samples"])))
    return n


@pytest.mark.parametrize("adj", list(ADJ))
def test_cfg1_assa_forward_adjoint_full(adj, monkeypatch):
    cfg = inputs.CONFIGS["cfg1"]
    c, s, op = cfg.centers(), cfg.sensors(), cfg.op_kwargs()
    ctx = make_ctx(c, s, op, monkeypatch=monkeypatch, adj=adj)
    p, kw = assa_kw(op)
    info = ctx.info()
    assert (info["assa"], info["assa_alpha"], info["assa_K"], info["assa_n_half"]) == (1, 2, 16, 8)
    assert info["adj_kernel"] == ADJ[adj][1], info
    x = inputs.dense_amplitudes(cfg.M)
    y = ctx.forward(T(x)).cpu().numpy()
    assert_parity(y, oracle.assa_forward(c, x, s, n_samples=op["n_samples"], **kw), "cfg1 assa forward")
    d = inputs.residual(cfg.n_sensors, cfg.n_samples)
    g = ctx.adjoint(T(d)).cpu().numpy()
    assert_parity(g, oracle.assa_adjoint(c, d, s, **kw), "cfg1 assa adjoint")
    assert ctx.count_pair_samples() == impulse_count(c, s, op, p["alpha"])


@pytest.mark.parametrize("adj", list(ADJ))
@pytest.mark.parametrize("seed", range(10))
def test_assa_random_suite(seed, adj, monkeypatch):
    c, s, op = inputs.random_suite_case(seed)
    rng = np.random.default_rng(seed)
    nmin = [25, 25, 9, 41, 25][seed % 5]
    ctx = make_ctx(c, s, op, nmin, monkeypatch=monkeypatch, adj=adj)
    assert ctx.info()["adj_kernel"] == ADJ[adj][1]
    p, kw = assa_kw(op, nmin)
    x = rng.random(c.shape[1]).astype(np.float32)
    y_ref = oracle.assa_forward(c, x, s, n_samples=op["n_samples"], **kw)
    if np.linalg.norm(y_ref) > 0:
        assert_parity(ctx.forward(T(x)).cpu().numpy(), y_ref, f"seed {seed} assa forward")
    d = rng.standard_normal((s.shape[1], op["n_samples"])).astype(np.float32)
    g_ref = oracle.assa_adjoint(c, d, s, **kw)
    if np.linalg.norm(g_ref) > 0:
        assert_parity(ctx.adjoint(T(d)).cpu().numpy(), g_ref, f"seed {seed} assa adjoint")
    assert ctx.count_pair_samples() == impulse_count(c, s, op, p["alpha"])


def test_assa_iterate_one_step():
    cfg = inputs.CONFIGS["cfg1"]
    c, s, op = cfg.centers(), cfg.sensors(), cfg.op_kwargs()
    ctx = make_ctx(c, s, op)
    p, kw = assa_kw(op)
    rng = np.random.default_rng(3)
    b = oracle.assa_forward(c, inputs.vessel_phantom(*cfg.grid), s, n_samples=op["n_samples"], **kw).astype(np.float32)
    z0 = rng.uniform(0.2, 0.9, cfg.M).astype(np.float32)
    zt, mt, vt = T(z0), torch.zeros(cfg.M, device=dev()), torch.zeros(cfg.M, device=dev())
    y_out = torch.empty((cfg.n_sensors, cfg.n_samples), device=dev())
    loss = torch.empty(1, device=dev())
    ctx.iterate(zt, mt, vt, T(b), lr=0.01, step=1, signals_out=y_out, loss_out=loss)
    torch.cuda.synchronize()
    geom = {"centers": c, "sensors": s, "op": op, "assa": {"alpha": p["alpha"], "K": p["K"]}}
    L_ref, gz_ref, y_ref = ir.loss_and_grad(z0.astype(np.float64), b.astype(np.float64), geom, ir.Hyper())
    assert_parity(y_out.cpu().numpy(), y_ref, "assa iterate signals")
    assert abs(loss.item() - L_ref) / L_ref <= 1e-5
    assert_parity(mt.cpu().numpy(), 0.1 * gz_ref, "assa iterate dL/dz")


def test_cfg4_assa_sampled():
    cfg = inputs.CONFIGS["cfg4"]
    c, s, op = cfg.centers(), cfg.sensors(), cfg.op_kwargs()
    ctx = make_ctx(c, s, op)
    p, kw = assa_kw(op)
    x = inputs.dense_amplitudes(cfg.M)
    y = ctx.forward(T(x)).cpu().numpy()
    rows = sample_rows(cfg.n_sensors)
    assert_parity(y[rows], oracle.assa_forward(c, x, s, n_samples=op["n_samples"], rows=rows, **kw), "cfg4 assa fwd")
    d = inputs.residual(cfg.n_sensors, cfg.n_samples)
    g = ctx.adjoint(T(d)).cpu().numpy()
    cols = sample_cols(cfg.M)
    assert_parity(g[cols], oracle.assa_adjoint(c, d, s, cols=cols, **kw), "cfg4 assa adj")
