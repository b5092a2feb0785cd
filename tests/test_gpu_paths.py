"""GPU parity of every forward / adjoint kernel path of the common configuration.

The bench configuration (degree-2 series, full windows of W = 16 samples)
runs the factorised-Gaussian forward (TAB) and the moment-polynomial adjoint
(k_adjoint_mp).  The other kernels of the same configuration -- the
lane-centred sensor-lane adjoint (k_adjoint_lcf), the TAB sensor-lane adjoint
(k_adjoint_t), the per-sample sensor-lane adjoint (k_adjoint_sl), the
lane-per-kernel adjoint (k_adjoint) and the per-sample-exponential forward --
are the fallbacks for contexts the fast kernels do not cover; the library
selects them at create time, and the environment switches GPAIR_NO_TAB /
GPAIR_ADJ_NO_MP / GPAIR_ADJ_NO_LCF / GPAIR_ADJ_NO_T force them here so each is
held to the same oracle gate (DESIGN.md sections 5, 6).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from oracle import ir  # noqa: E402
from paper_2602_03893_b200 import gpair, inputs  # noqa: E402
from tests_common import T, assert_parity, assert_state_update  # noqa: E402

pytestmark = pytest.mark.gpu

# switches -> (info.tab, info.adj_kernel)
PATHS = {
    "tab+mp": ({}, (1, 4)),
    "tab+mp48": ({"GPAIR_MP_ROW48": "1"}, (1, 4)),  # the 48-B (degree-7) moment rows
    "tab+lcf": ({"GPAIR_ADJ_NO_MP": "1"}, (1, 2)),
    "tab+lane_t": ({"GPAIR_ADJ_NO_MP": "1", "GPAIR_ADJ_NO_LCF": "1"}, (1, 1)),
    "tab+lane_kernel": ({"GPAIR_ADJ_NO_MP": "1", "GPAIR_ADJ_NO_LCF": "1", "GPAIR_ADJ_NO_T": "1"}, (1, 0)),
    "per_sample_exp+mp": ({"GPAIR_NO_TAB": "1"}, (0, 4)),
    "per_sample_exp+lane_sl": ({"GPAIR_NO_TAB": "1", "GPAIR_ADJ_NO_MP": "1"}, (0, 3)),
    "per_sample_exp+lane_kernel": ({"GPAIR_NO_TAB": "1", "GPAIR_ADJ_NO_MP": "1", "GPAIR_ADJ_NO_T": "1"}, (0, 0)),
    # sensor-group pipeline of gpair_iterate (opt-in): forward / reducer / adjoint per 256-sensor group
    "tab+mp+pipeline": ({"GPAIR_PIPELINE": "1"}, (1, 4)),
    "tab+lcf+pipeline": ({"GPAIR_PIPELINE": "1", "GPAIR_ADJ_NO_MP": "1"}, (1, 2)),
    "per_sample_exp+lane_sl+pipeline": ({"GPAIR_NO_TAB": "1", "GPAIR_PIPELINE": "1", "GPAIR_ADJ_NO_MP": "1"}, (0, 3)),
    # register-window forward (opt-in)
    "tab_union+mp": ({"GPAIR_FWD_UNION": "1"}, (1, 4)),
}
ENV_KEYS = ("GPAIR_NO_TAB", "GPAIR_MP_ROW48", "GPAIR_ADJ_NO_MP", "GPAIR_ADJ_NO_LCF", "GPAIR_ADJ_NO_T", "GPAIR_PIPELINE", "GPAIR_FWD_UNION")


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_03893_b200 import build

    build.build()


check = assert_parity


def small_tab_case():
    """TAB-eligible and oracle-cheap: 16^3 kernels at dx = sigma = 0.1 mm, 64-sensor
    R = 60 mm hemisphere, 2048 samples at 40 MHz (W = 16, degree-2 series)."""
    c = inputs.grid_centers(16, 16, 16, 1e-4)
    s = inputs.hemisphere(64, 60e-3)
    op = dict(sigma=1e-4, v=1500.0, fs=40e6, n_samples=2048, t0=0.0, k=3.0)
    return c, s, op


def make_ctx(c, s, op, monkeypatch, env):
    for key in ENV_KEYS:
        monkeypatch.delenv(key, raising=False)
    for key, val in env.items():
        monkeypatch.setenv(key, val)
    return gpair.Context(T(c), T(s), sigma=op["sigma"], v=op["v"], fs=op["fs"], n_samples=op["n_samples"],
                         t0=op["t0"], k=op["k"])


@pytest.mark.parametrize("path", list(PATHS))
def test_forward_adjoint_each_path(path, monkeypatch):
    env, expect = PATHS[path]
    c, s, op = small_tab_case()
    ctx = make_ctx(c, s, op, monkeypatch, env)
    info = ctx.info()
    assert (info["tab"], info["adj_kernel"]) == expect, info
    assert info["fwd_union"] == (1 if env.get("GPAIR_FWD_UNION") == "1" else 0), info
    x = inputs.dense_amplitudes(c.shape[1])
    check(ctx.forward(T(x)).cpu().numpy(), oracle.forward(c, x, s, **op), f"{path} forward")
    d = inputs.residual(s.shape[1], op["n_samples"])
    akw = {k: v for k, v in op.items() if k != "n_samples"}
    check(ctx.adjoint(T(d)).cpu().numpy(), oracle.adjoint(c, d, s, **akw), f"{path} adjoint")
    ctx.close()


@pytest.mark.parametrize("path", list(PATHS))
@pytest.mark.parametrize("mode", [0, 1])
def test_iterate_each_path_teacher_forced(path, mode, monkeypatch):
    """One Algorithm-2 iteration (NPC + Adam, or the clamp step) from an oracle
    state through each adjoint kernel and its update epilogue."""
    env, _ = PATHS[path]
    c, s, op = small_tab_case()
    M = c.shape[1]
    ctx = make_ctx(c, s, op, monkeypatch, env)
    rng = np.random.default_rng(17)
    x_true = inputs.vessel_phantom(16, 16, 16) + 0.1 * rng.random(M).astype(np.float32)
    b = oracle.forward(c, x_true, s, **op).astype(np.float32)
    z0 = rng.uniform(0.2, 0.9, M).astype(np.float32)
    geom = {"centers": c, "sensors": s, "op": op}
    hp = ir.Hyper(mode="npc" if mode == 0 else "clamp")
    _, gz0, _ = ir.loss_and_grad(z0.astype(np.float64), b.astype(np.float64), geom, hp)
    m0 = (0.5 * gz0 * rng.uniform(0.5, 1.5, M)).astype(np.float32)
    v0 = (gz0 * gz0 * rng.uniform(0.5, 1.5, M)).astype(np.float32)
    t_step = 5
    lr = gpair.cawr_lr(t_step - 1, 1e-4, 0.1, 50, 1)
    zt, mt, vt = T(z0), T(m0), T(v0)
    loss = torch.empty(1, device="cuda")
    ctx.iterate(zt, mt, vt, T(b), lr=lr, step=t_step, mode=mode, loss_out=loss)
    torch.cuda.synchronize()
    L_ref, gz_ref, _ = ir.loss_and_grad(z0.astype(np.float64), b.astype(np.float64), geom, hp)
    assert abs(loss.item() - L_ref) / L_ref <= 1e-5
    if mode == 0:
        z_ref, m_ref, v_ref = ir.adam_update(z0.astype(np.float64), m0.astype(np.float64), v0.astype(np.float64),
                                             gz_ref, lr, t_step, hp)
        check(mt.cpu().numpy() - 0.9 * m0, m_ref - 0.9 * m0, f"{path} Adam m increment")
        check(vt.cpu().numpy(), v_ref, f"{path} Adam v")
        assert_state_update(zt.cpu().numpy(), z0, z_ref, f"{path} Adam z step")
    else:
        assert_state_update(zt.cpu().numpy(), z0, np.maximum(z0 - lr * gz_ref, 0.0), f"{path} clamp step")
    ctx.close()


def test_bench_configuration_uses_fast_paths(monkeypatch):
    """cfg2 / cfg4 geometry (the bench's) selects the TAB forward and the moment-polynomial adjoint."""
    for key in ENV_KEYS:
        monkeypatch.delenv(key, raising=False)
    cfg = inputs.CONFIGS["cfg2"]
    ctx = gpair.Context(T(cfg.centers()), T(cfg.sensors()), sigma=cfg.sig, v=cfg.v, fs=cfg.fs,
                        n_samples=cfg.n_samples, t0=cfg.t0, k=cfg.k)
    info = ctx.info()
    assert info["tab"] == 1 and info["adj_kernel"] == 4, info
    ctx.close()


# randomized geometries on the fast paths: W in {12, 16, 20, 24, 32} (sigma = W h / 6), grid or
# jittered (non-grid sort) kernels, hemisphere or planar arrays, t0 > 0 and records that clip
@pytest.mark.parametrize("seed", range(10))
def test_fast_paths_random_geometry(seed, monkeypatch):
    rng = np.random.default_rng(1000 + seed)
    W = int(rng.choice([12, 16, 20, 24, 32]))
    fs, v = 40e6, 1500.0
    sigma = W * (v / fs) / 6.0
    n = rng.integers(5, 13, size=3)
    c = inputs.grid_centers(int(n[0]), int(n[1]), int(n[2]), sigma, jitter=0.4 if seed % 3 == 0 else 0.0, seed=seed)
    if seed % 4 == 3:
        s = inputs.planar_checkerboard(n_side=8, pitch=6e-3, z=-30e-3)
    else:
        s = inputs.hemisphere(int(rng.integers(20, 70)), float(rng.uniform(40e-3, 80e-3)))
    t0 = float(rng.uniform(0.0, 15e-6))
    rmax = float(np.max(np.linalg.norm(s[:, :, None] - c[:, None, :].mean(axis=2, keepdims=True), axis=0)))
    n_samples = int((rmax / v - t0) * fs) + int(rng.integers(-8, 24))  # some windows reach past the record
    op = dict(sigma=sigma, v=v, fs=fs, n_samples=n_samples, t0=t0, k=3.0)
    # even seeds: the moment-polynomial adjoint; odd seeds: the lane-centred one
    ctx = make_ctx(c, s, op, monkeypatch, {} if seed % 2 == 0 else {"GPAIR_ADJ_NO_MP": "1"})
    info = ctx.info()
    assert info["adj_kernel"] == (4 if seed % 2 == 0 else 2), info
    x = rng.random(c.shape[1]).astype(np.float32)
    check(ctx.forward(T(x)).cpu().numpy(), oracle.forward(c, x, s, **op), f"seed {seed} W {W} forward")
    d = rng.standard_normal((s.shape[1], n_samples)).astype(np.float32)
    akw = {k: v for k, v in op.items() if k != "n_samples"}
    check(ctx.adjoint(T(d)).cpu().numpy(), oracle.adjoint(c, d, s, **akw), f"seed {seed} W {W} adjoint")
    assert info["tab"] == 1, info  # every case is on the fast (TAB) path
    ctx.close()


# window lengths outside the TAB range (W = 5 of cfg4', W = 8, W = 48 / 64 of desk-like sigma):
# the per-sample sensor-lane adjoint (k_adjoint_sl) and the per-sample forward
@pytest.mark.parametrize("W", [5, 8, 48, 64])
def test_per_sample_sensor_lane_adjoint(W, monkeypatch):
    fs, v = 40e6, 1500.0
    sigma = W * (v / fs) / 6.0
    c = inputs.grid_centers(10, 9, 8, sigma)
    s = inputs.hemisphere(48, 60e-3)
    op = dict(sigma=sigma, v=v, fs=fs, n_samples=1900 + 2 * W, t0=2e-6, k=3.0)
    ctx = make_ctx(c, s, op, monkeypatch, {"GPAIR_ADJ_NO_MP": "1"})
    info = ctx.info()
    assert info["adj_kernel"] == 3 and info["tab"] == 0, info
    rng = np.random.default_rng(W)
    x = rng.random(c.shape[1]).astype(np.float32)
    check(ctx.forward(T(x)).cpu().numpy(), oracle.forward(c, x, s, **op), f"W {W} forward")
    d = rng.standard_normal((s.shape[1], op["n_samples"])).astype(np.float32)
    akw = {k: v for k, v in op.items() if k != "n_samples"}
    check(ctx.adjoint(T(d)).cpu().numpy(), oracle.adjoint(c, d, s, **akw), f"W {W} adjoint")
    ctx.close()


# the moment-polynomial adjoint's eligibility boundary: any exact-integer window whose
# degree-7 interpolant of the window weights reaches 1e-8 of max |f|, i.e. W >= 10 at k = 3 (sigma >=
# 1.67 samples), including window lengths that are not the forward's template sizes (10, 13); W = 8
# falls back to the sensor-lane per-sample adjoint.  Record clipping at both ends (the record starts
# inside the nearest windows and ends inside the farthest).  Jittered (non-grid) kernels below W = 40
# (wide windows over a jittered cloud need more staged rows than the ring holds: fallback kernel).
@pytest.mark.parametrize("W", [8, 10, 13, 20, 64])
def test_moment_adjoint_window_lengths(W, monkeypatch):
    fs, v = 40e6, 1500.0
    sigma = W * (v / fs) / 6.0
    c = inputs.grid_centers(9, 10, 8, sigma, jitter=0.3 if W < 40 else 0.0, seed=W)
    s = inputs.hemisphere(40, 50e-3)
    # the record starts inside the nearest windows and ends inside the farthest ones
    half = 0.5 * float(np.max(c.max(axis=1) - c.min(axis=1)))
    t0 = (50e-3 - 0.8 * half) / v
    op = dict(sigma=sigma, v=v, fs=fs, n_samples=int(1.6 * half / v * fs) + W, t0=t0, k=3.0)
    ctx = make_ctx(c, s, op, monkeypatch, {})
    info = ctx.info()
    assert info["adj_kernel"] == (3 if W < 10 else 4), info
    assert (info["adj_fit_err"] <= 1e-8) == (W >= 10), info
    rng = np.random.default_rng(100 + W)
    d = rng.standard_normal((s.shape[1], op["n_samples"])).astype(np.float32)
    akw = {k: v for k, v in op.items() if k != "n_samples"}
    check(ctx.adjoint(T(d)).cpu().numpy(), oracle.adjoint(c, d, s, **akw), f"W {W} adjoint")
    ctx.close()


# any window length (fast packed paths where W is a template size, generic paths otherwise),
# degree-2 or degree-5 series (array radius), jitter, t0 > 0, clipped records
@pytest.mark.parametrize("seed", range(8))
def test_random_geometry_any_window(seed, monkeypatch):
    rng = np.random.default_rng(2000 + seed)
    W = int([5, 6, 7, 8, 9, 10, 13, 40][seed])
    fs, v = float(rng.choice([20e6, 40e6])), 1500.0
    sigma = W * (v / fs) / 6.0
    n = rng.integers(4, 10, size=3)
    c = inputs.grid_centers(int(n[0]), int(n[1]), int(n[2]), sigma, jitter=0.3 if seed % 2 else 0.0, seed=seed)
    s = inputs.hemisphere(int(rng.integers(16, 48)), float(rng.uniform(15e-3, 70e-3)))
    t0 = float(rng.uniform(0.0, 5e-6))
    rmax = float(np.max(np.linalg.norm(s[:, :, None] - c[:, None, :].mean(axis=2, keepdims=True), axis=0)))
    n_samples = int((rmax / v - t0) * fs) + int(rng.integers(-4, 16))
    op = dict(sigma=sigma, v=v, fs=fs, n_samples=n_samples, t0=t0, k=3.0)
    ctx = make_ctx(c, s, op, monkeypatch, {})
    x = rng.random(c.shape[1]).astype(np.float32)
    check(ctx.forward(T(x)).cpu().numpy(), oracle.forward(c, x, s, **op), f"seed {seed} W {W} forward")
    d = rng.standard_normal((s.shape[1], n_samples)).astype(np.float32)
    akw = {k: v for k, v in op.items() if k != "n_samples"}
    check(ctx.adjoint(T(d)).cpu().numpy(), oracle.adjoint(c, d, s, **akw), f"seed {seed} W {W} adjoint")
    ctx.close()


@pytest.mark.parametrize("pipeline", ["0", "1"])
def test_iterate_cuda_graph_capture(pipeline, monkeypatch):
    """gpair_iterate is asynchronous on the caller's stream and capturable in a CUDA graph
    (with the opt-in sensor-group pipeline too: fork/join through events); replaying the
    graph gives bit-identical state to eager calls."""
    monkeypatch.setenv("GPAIR_PIPELINE", pipeline)
    c, s, op = small_tab_case()
    M = c.shape[1]
    ctx = gpair.Context(T(c), T(s), sigma=op["sigma"], v=op["v"], fs=op["fs"], n_samples=op["n_samples"],
                        t0=op["t0"], k=op["k"])
    rng = np.random.default_rng(5)
    b = T(oracle.forward(c, rng.random(M).astype(np.float32), s, **op).astype(np.float32))
    z0 = rng.uniform(0.2, 0.9, M).astype(np.float32)

    def run(use_graph):
        z, m, v = T(z0), torch.zeros(M, device="cuda"), torch.zeros(M, device="cuda")
        loss = torch.zeros(1, device="cuda")
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            ctx.iterate(z, m, v, b, lr=0.01, step=1, loss_out=loss, stream=st)  # warm-up / first step
            if use_graph:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=st):
                    ctx.iterate(z, m, v, b, lr=0.01, step=2, loss_out=loss, stream=st)
                for _ in range(3):
                    g.replay()
            else:
                for _ in range(3):
                    ctx.iterate(z, m, v, b, lr=0.01, step=2, loss_out=loss, stream=st)
        torch.cuda.synchronize()
        return z.cpu().numpy(), loss.cpu().numpy()

    ze, le = run(False)
    zg, lg = run(True)
    assert np.array_equal(ze, zg) and np.array_equal(le, lg)
    ctx.close()
