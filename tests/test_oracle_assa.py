"""Pins of the fp64 ASSA oracle (Eqs. 8-17,
Algorithm 1).  Expected values come from hand evaluation of Eq. 8
and Eq. 9 (SPEC examples S:80-81), the closed-form F2 matrix
(every pair's taps written out directly, a different algorithm from the
three-stage pipeline), the dot test, the taps' odd symmetry, and convergence
to the direct operator (pinned in test_oracle_pins.py) as alpha grows."""
import math

import numpy as np
import pytest

import oracle
from paper_2602_03893_b200 import inputs

V = 1500.0


def test_assa_params_examples():
    """Eq. 8 hand values (Fig. 1f: f_s = 20 MHz -> 80 MHz)."""
    p = oracle.assa_params(62.5e-6, V, 20e6)
    assert (p["n_half"], p["alpha"], p["K"], p["fs_up"]) == (3, 4, 12, 80e6)
    p = oracle.assa_params(0.2e-3, V, 20e6)
    assert (p["n_half"], p["alpha"]) == (8, 2)
    p = oracle.assa_params(1e-4, V, 40e6)  # the bench constants
    assert (p["n_half"], p["alpha"], p["K"], p["fs_up"]) == (8, 2, 16, 80e6)
    assert oracle.assa_params(1e-3, V, 40e6)["alpha"] == 1  # N_half >= 12 -> no upsampling


def test_assa_index_examples():
    """Eq. 9: k = floor(r/v f_s^up + 0.5)."""
    c = np.zeros((3, 1), np.float32)
    K = 16
    # r = 37.5 mm at 80 MHz -> k = 2000: the single impulse's taps land around alpha n = 2000
    s = np.array([[0.0], [0.0], [-0.0375]], np.float32)
    y = oracle.assa_forward(c, [1.0], s, sigma=1e-4, v=V, fs=40e6, n_samples=1100, alpha=2, K=K)[0]
    h = oracle.assa_taps(1e-4, V, 80e6, K)
    r = float(np.float32(-0.0375)) * -1
    assert math.floor(r / V * 80e6 + 0.5) == 2000  # r = fp32(37.5 mm)
    # y[n] = h[2n - 2000] / r for |2n - 2000| <= K
    for n in range(990, 1010):
        kk = 2 * n - 2000
        exp = h[kk + K] / r if abs(kk) <= K else 0.0
        assert y[n] == pytest.approx(exp, rel=1e-13, abs=1e-18)
    # round half up: r/v f_s^up = 10.5 -> 11
    assert math.floor(10.5 + 0.5) == 11


def test_taps_odd_and_zero_center():
    """h[0] = 0 and h[-k] = -h[k] exactly; sum of taps = 0."""
    for sigma, fs in [(1e-4, 40e6), (62.5e-6, 20e6), (0.2e-3, 20e6)]:
        p = oracle.assa_params(sigma, V, fs)
        h = oracle.assa_taps(sigma, V, p["fs_up"], p["K"])
        K = p["K"]
        assert h[K] == 0.0
        assert np.array_equal(h[K + 1:], -h[:K][::-1])
        assert abs(h.sum()) <= 1e-12 * np.abs(h).max()
        # edge tap: |d[K]| = v K dt_up >= 3 sigma
        assert V * K / p["fs_up"] >= 3 * sigma * (1 - 1e-12)


def _f2_matrix(c, s, sigma, v, fs, n_samples, alpha, K, t0):
    """Closed-form F2 entries: A[(j,n), i] = h[alpha n - k_ij] / r_ij
    for |alpha n - k_ij| <= K and k_ij in [0, alpha N_t)."""
    fs_up = alpha * fs
    h = oracle.assa_taps(sigma, v, fs_up, K)
    c64, s64 = c.astype(np.float64), s.astype(np.float64)
    M, Nd = c.shape[1], s.shape[1]
    A = np.zeros((Nd * n_samples, M))
    for j in range(Nd):
        for i in range(M):
            d = c64[:, i] - s64[:, j]
            r = math.sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2])
            kij = math.floor((r / v - t0) * fs_up + 0.5)
            if not (0 <= kij < alpha * n_samples):
                continue
            for n in range(n_samples):
                q = alpha * n - kij
                if abs(q) <= K:
                    A[j * n_samples + n, i] = h[q + K] / r
    return A


@pytest.mark.parametrize("seed,fs,sigma", [(0, 40e6, 1e-4), (1, 20e6, 62.5e-6), (2, 50e6, 0.12e-3)])
def test_assa_pipeline_equals_f2_matrix(seed, fs, sigma):
    rng = np.random.default_rng(seed)
    c = inputs.grid_centers(3, 3, 2, 1e-4, jitter=0.4, seed=seed)
    s = inputs.hemisphere(5, 0.011)
    t0 = 0.4e-6 * seed
    n_samples = int((0.0116 / V - t0) * fs)  # short record: some impulses fall outside
    p = oracle.assa_params(sigma, V, fs)
    A = _f2_matrix(c, s, sigma, V, fs, n_samples, p["alpha"], p["K"], t0)
    x = rng.standard_normal(c.shape[1])
    d = rng.standard_normal((s.shape[1], n_samples))
    kw = dict(sigma=sigma, v=V, fs=fs, alpha=p["alpha"], K=p["K"], t0=t0)
    y = oracle.assa_forward(c, x, s, n_samples=n_samples, **kw)
    g = oracle.assa_adjoint(c, d, s, **kw)
    assert np.linalg.norm(y.ravel() - A @ x) <= 1e-12 * np.linalg.norm(A @ x)
    assert np.linalg.norm(g - A.T @ d.ravel()) <= 1e-12 * np.linalg.norm(A.T @ d.ravel())


@pytest.mark.parametrize("seed", range(6))
def test_assa_dot_test(seed):
    c, s, op = inputs.random_suite_case(seed)
    p = oracle.assa_params(op["sigma"], op["v"], op["fs"])
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(c.shape[1])
    d = rng.standard_normal((s.shape[1], op["n_samples"]))
    kw = dict(sigma=op["sigma"], v=op["v"], fs=op["fs"], alpha=p["alpha"], K=p["K"], t0=op["t0"])
    Ax = oracle.assa_forward(c, x, s, n_samples=op["n_samples"], **kw)
    ATd = oracle.assa_adjoint(c, d, s, **kw)
    lhs, rhs = float(np.sum(Ax * d)), float(np.dot(x, ATd))
    assert abs(lhs - rhs) <= 1e-10 * np.linalg.norm(Ax) * np.linalg.norm(d)


def test_assa_converges_to_direct_operator():
    """ASSA's alignment error shrinks as alpha grows: the
    relative L2 distance to the direct operator falls roughly as 1/alpha."""
    cfg = inputs.CONFIGS["cfg1"]
    c, s, op = cfg.centers(), cfg.sensors(), cfg.op_kwargs()
    x = inputs.dense_amplitudes(cfg.M)
    y_direct = oracle.forward(c, x, s, **op)
    errs = []
    for alpha in (1, 2, 4, 8, 16):
        y = oracle.assa_forward(c, x, s, sigma=op["sigma"], v=op["v"], fs=op["fs"], n_samples=op["n_samples"],
                                alpha=alpha, K=8 * alpha, t0=op["t0"])
        errs.append(np.linalg.norm(y - y_direct) / np.linalg.norm(y_direct))
    assert all(a > b for a, b in zip(errs, errs[1:])), errs
    assert errs[-1] < 0.25 * errs[1] and errs[-1] < 0.02, errs
