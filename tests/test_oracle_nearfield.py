"""Pins of the row-f4 oracle extensions: the near-field
operator (Eq. 6 with both terms, readings N1-N3) and
per-kernel sigma_i (reading N2).  Expected values come from Poisson's
formula by quadrature (the P1 helper), the closed-form r -> 0 limit of
Eq. 6, a brute-force loop over every sample, superposition of single-kernel
scalar-sigma calls, and the dot test; none re-calls the function under test
to make its own expected value.
"""
import math

import numpy as np
import pytest

import oracle
from paper_2602_03893_b200 import inputs
from test_oracle_pins import _poisson_quadrature

V = 1500.0
SIG = 1e-4


def _one_pair(r, fs=200e6, n_samples=64, t0=0.0, k=12.0, sigma=SIG):
    c = np.zeros((3, 1), np.float32)
    s = np.array([[r], [0.0], [0.0]], np.float32)
    return c, s, dict(sigma=sigma, v=V, fs=fs, n_samples=n_samples, t0=t0, k=k)


@pytest.mark.parametrize("r_over_sigma", [0.3, 1.0, 2.0, 2.9, 4.5])
def test_nf_single_pair_matches_poisson_quadrature(r_over_sigma):
    """Near field (r comparable with sigma): the two-term operator equals the
    quadrature of Poisson's solution (Eq. 3) at every sample; k = 12
    makes the truncation invisible (e^-72)."""
    c, s, op = _one_pair(r_over_sigma * SIG)
    A = 1.3
    y = oracle.forward(c, np.array([A]), s, near_field=True, **op)[0]
    r = float(np.float32(r_over_sigma * SIG))
    peak = A * 1.0  # |p| <= A near the source (Eq. 6 at r -> 0, t = 0)
    worst = 0.0
    for n in range(1, op["n_samples"]):
        t = n / op["fs"]
        worst = max(worst, abs(y[n] - _poisson_quadrature(A, r, t, V, SIG)) / peak)
    assert worst <= 1e-10, worst


def test_nf_limit_r_to_zero():
    """Eq. 6 as r -> 0 (l'Hopital): p -> A (1 - tau^2/sigma^2) exp(-tau^2 / 2 sigma^2),
    tau = v t.  At r = 1e-6 sigma the O(r^2) remainder is 1e-12."""
    c, s, op = _one_pair(1e-6 * SIG)
    A = 0.7
    y = oracle.forward(c, np.array([A]), s, near_field=True, **op)[0]
    for n in range(op["n_samples"]):
        tau = V * n / op["fs"]
        lim = A * (1.0 - tau * tau / SIG ** 2) * math.exp(-tau * tau / (2 * SIG ** 2))
        assert abs(y[n] - lim) <= 1e-8 * A, (n, y[n], lim)


def test_nf_far_pairs_bitwise_equal_to_outgoing():
    """Every pair far (r > k sigma, t0 >= 0): the incoming window is empty and
    the near-field operator is the Eq. 7 operator bit for bit."""
    for seed in range(4):
        c, s, op = inputs.random_suite_case(seed)
        M = c.shape[1]
        x = np.random.default_rng(seed).random(M)
        np.testing.assert_array_equal(oracle.forward(c, x, s, near_field=True, **op), oracle.forward(c, x, s, **op))
        d = inputs.residual(s.shape[1], op["n_samples"], seed=seed)
        kw = {k: v for k, v in op.items() if k != "n_samples"}
        np.testing.assert_array_equal(oracle.adjoint(c, d, s, near_field=True, **kw), oracle.adjoint(c, d, s, **kw))


def _near_geometry(seed):
    """Sensors inside and around a small kernel grid (near pairs everywhere)."""
    rng = np.random.default_rng(seed)
    c = inputs.grid_centers(4, 3, 3, 1e-4, jitter=0.3, seed=seed)
    s = rng.uniform(-4e-4, 4e-4, (3, 7)).astype(np.float32)
    sig = rng.uniform(0.6, 1.4, c.shape[1]) * SIG
    sig = sig.astype(np.float32).astype(np.float64)
    op = dict(sigma=SIG, v=V, fs=40e6, n_samples=40, t0=float(rng.uniform(-1e-7, 1e-7)), k=3.0)
    return c, s, sig, op


def _brute(c, s, amp, sig, op):
    """Every (i, j, n) with no candidate ranges: Eq. 6, each term truncated."""
    M, Nd, Nt = c.shape[1], s.shape[1], op["n_samples"]
    y = np.zeros((Nd, Nt))
    cd, sd = c.astype(np.float64), s.astype(np.float64)
    for j in range(Nd):
        for i in range(M):
            r = math.sqrt(sum((cd[a, i] - sd[a, j]) ** 2 for a in range(3)))
            ks = op["k"] * sig[i]
            for n in range(Nt):
                t = op["t0"] + n / op["fs"]
                tot = 0.0
                for d in (r - V * t, r + V * t):
                    if abs(d) < ks:
                        tot += d * math.exp(-d * d / (2 * sig[i] ** 2))
                y[j, n] += amp[i] * tot / (2 * r)
    return y


@pytest.mark.parametrize("seed", [0, 1])
def test_nf_sigmas_brute_force_and_dot_test(seed):
    c, s, sig, op = _near_geometry(seed)
    M, Nd = c.shape[1], s.shape[1]
    x = np.random.default_rng(seed + 5).standard_normal(M)
    y = oracle.forward(c, x, s, sigmas=sig, near_field=True, **op)
    yb = _brute(c, s, x, sig, op)
    assert np.max(np.abs(y - yb)) <= 1e-12 * np.max(np.abs(yb))
    d = np.random.default_rng(seed + 9).standard_normal((Nd, op["n_samples"]))
    kw = {k: v for k, v in op.items() if k != "n_samples"}
    g = oracle.adjoint(c, d, s, sigmas=sig, near_field=True, **kw)
    lhs, rhs = float(np.sum(y * d)), float(np.dot(x, g))
    assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(y) * np.linalg.norm(d)


def test_sigmas_superposition_of_single_kernels():
    """sigma_i is applied to kernel i: the multi-kernel operator is the sum of
    single-kernel scalar-sigma operators (Eq. 2 linearity)."""
    cfg = inputs.CONFIGS["cfg1"]
    c, s, op = cfg.centers(), cfg.sensors(), cfg.op_kwargs()
    rng = np.random.default_rng(3)
    M = c.shape[1]
    sig = (rng.uniform(0.5, 1.5, M) * op["sigma"]).astype(np.float32).astype(np.float64)
    x = rng.random(M)
    pick = rng.choice(M, 24, replace=False)
    xs = np.zeros(M)
    xs[pick] = x[pick]
    y = oracle.forward(c, xs, s, sigmas=sig, **op)
    ys = np.zeros_like(y)
    for i in pick:
        ys += oracle.forward(c[:, i:i + 1], x[i:i + 1], s, **dict(op, sigma=sig[i]))
    assert np.max(np.abs(y - ys)) <= 1e-13 * np.max(np.abs(ys))
    d = inputs.residual(s.shape[1], op["n_samples"])
    kw = {k: v for k, v in op.items() if k != "n_samples"}
    g = oracle.adjoint(c, d, s, sigmas=sig, cols=pick, **kw)
    for q, i in enumerate(pick):
        gi = oracle.adjoint(c[:, i:i + 1], d, s, **dict(kw, sigma=sig[i]))[0]
        assert g[q] == gi


def test_sigmas_all_equal_is_scalar_path():
    cfg = inputs.CONFIGS["cfg1"]
    c, s, op = cfg.centers(), cfg.sensors(), cfg.op_kwargs()
    x = inputs.dense_amplitudes(c.shape[1])
    sig = np.full(c.shape[1], op["sigma"])
    np.testing.assert_array_equal(oracle.forward(c, x, s, sigmas=sig, **op), oracle.forward(c, x, s, **op))


def test_nf_r_zero_is_geometry_error():
    c, s, op = _one_pair(0.0)
    with pytest.raises(oracle.OracleGeometryError):
        oracle.forward(c, np.ones(1), s, near_field=True, **op)
