"""CPU pin of the moment-polynomial adjoint's reformulation, in fp64 numpy.

The GPU adjoint k_adjoint_mp evaluates Eq. 7's adjoint (transposed as in
P:357-389) as g_i = sum_j w_ij sum_k xi_ij^k M_k[j][n_lo(i,j)], with the moments of the residual
M_k[j][n] = sum_m c_mk delta_j[n + m] (delta = 0 outside the record) and c_mk the Chebyshev
interpolants of the window weights f(xi0 + xi - m), f(u) = u 2^{K u^2}.  This test restates that
algebra independently of the GPU code (plain numpy, fp64 throughout) and checks it against the
fp64 oracle's direct enumeration: the two agree to the interpolation error (~1e-10 at degree 7,
~4e-9 at degree 6), including windows clipped by both ends of the record.  It pins the method,
not the kernel; the kernel is held to the oracle by the -m gpu tests.
"""
import math

import numpy as np
import pytest

import oracle
from paper_2602_03893_b200 import inputs


def chebyshev_fit(W, K, deg):
    """c[m][k]: interpolant of f(xi0 + xi - m) at the deg + 1 Chebyshev nodes of [-1/2, 1/2]."""
    P = deg + 1
    xi0 = 0.5 * W - 0.5
    nodes = 0.5 * np.cos((2 * np.arange(P) + 1) * math.pi / (2 * P))
    V = np.vander(nodes, P, increasing=True)
    f = lambda u: u * np.exp2(K * u * u)  # noqa: E731
    return np.array([np.linalg.solve(V, f(xi0 + nodes - m)) for m in range(W)])


def moment_adjoint(c, delta, s, *, sigma, v, fs, t0, k, deg):
    """g via per-pair (n_lo, xi, w) and the residual's moments, fp64."""
    h = v / fs
    ku = k * sigma / h
    W = int(round(2 * ku))
    assert abs(2 * ku - W) < 1e-9, "the reformulation needs an integer window length"
    K = -math.log2(math.e) * h * h / (2 * sigma * sigma)
    coef = chebyshev_fit(W, K, deg)  # [W][P]
    Nd, Nt = delta.shape
    # M[j][n + W - 1][k] for start samples n in [-(W - 1), Nt - 1] (zero-padded delta)
    dpad = np.concatenate([np.zeros((Nd, W - 1)), delta.astype(np.float64), np.zeros((Nd, W - 1))], axis=1)
    M = np.zeros((Nd, Nt + W - 1, coef.shape[1]))
    for m in range(W):
        M += dpad[:, m:m + Nt + W - 1, None] * coef[m][None, None, :]
    g = np.zeros(c.shape[1])
    c64, s64 = c.astype(np.float64), s.astype(np.float64)
    for j in range(Nd):
        d = c64 - s64[:, j:j + 1]
        r = np.sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2])
        e = (r / v - t0) * fs  # continuous sample position of r
        n_lo = np.floor(e - ku).astype(np.int64) + 1  # first n with |e - n| < ku
        xi = (e - n_lo) - (ku - 0.5)
        w = h / (2.0 * r)
        row = n_lo + W - 1
        ok = (row >= 0) & (row < Nt + W - 1)  # windows entirely outside the record contribute 0
        Mk = np.zeros((c.shape[1], coef.shape[1]))
        Mk[ok] = M[j, row[ok]]
        poly = np.zeros(c.shape[1])
        for kk in range(coef.shape[1] - 1, -1, -1):
            poly = poly * xi + Mk[:, kk]
        g += w * poly
    return g


@pytest.mark.parametrize("deg,tol", [(7, 1e-9), (6, 2e-8)])
def test_moment_reformulation_matches_the_direct_adjoint(deg, tol):
    # W = 16 samples (sigma = dx = 0.1 mm at 40 MHz); a short record that starts inside the nearest
    # windows and ends inside the farthest ones, so both record edges clip
    c = inputs.grid_centers(6, 5, 4, 1e-4, jitter=0.3, seed=3)
    s = inputs.hemisphere(24, 20e-3)
    v, fs, sigma = 1500.0, 40e6, 1e-4
    t0 = (20e-3 - 0.4e-3) / v
    Nt = int(0.8e-3 / v * fs) + 16
    rng = np.random.default_rng(11)
    delta = rng.standard_normal((s.shape[1], Nt)).astype(np.float32)
    ref = oracle.adjoint(c, delta, s, sigma=sigma, v=v, fs=fs, t0=t0, k=3.0)
    got = moment_adjoint(c, delta, s, sigma=sigma, v=v, fs=fs, t0=t0, k=3.0, deg=deg)
    err = np.abs(got - ref).max() / np.abs(ref).max()
    assert err <= tol, err


def test_moment_fit_error_bounds():
    # the create-time acceptance rule (max interpolation error <= 1e-8 of max |f|) at k = 3:
    # W = 16 passes at degree 6 and 7, W = 8 fails at degree 7 (falls back to another kernel)
    def fit_err(W, deg):
        h = 1.0
        sigma = W * h / 6.0
        K = -math.log2(math.e) * h * h / (2 * sigma * sigma)
        coef = chebyshev_fit(W, K, deg)
        xs = np.linspace(-0.5, 0.5, 4001)
        xi0 = 0.5 * W - 0.5
        f = lambda u: u * np.exp2(K * u * u)  # noqa: E731
        errs = [np.abs(np.polynomial.polynomial.polyval(xs, coef[m]) - f(xi0 + xs - m)).max() for m in range(W)]
        fmax = max(np.abs(f(xi0 + xs - m)).max() for m in range(W))
        return max(errs) / fmax
    assert fit_err(16, 7) < 1e-9
    assert fit_err(16, 6) < 1e-8
    assert fit_err(8, 7) > 1e-8
