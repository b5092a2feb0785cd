"""Pins of the fp64 oracle against what the paper and mathematics fix.

Each test names the pin of SURVEY.md 8(c) it implements and the PAPER.md
passage it follows.  None of them re-calls the oracle to produce its own
expected value: expected values come from Poisson's formula by quadrature,
hand-derived closed forms (tests/golden/known_values.txt), a brute-force loop
over ALL samples, the dense matrix of the operator, or finite differences.
"""
import math

import numpy as np
import pytest

import oracle
from oracle import ir
from paper_2602_03893_b200 import inputs

V = 1500.0
SIG = 1e-4


# ---------------------------------------------------------------- P1 ---------
def _poisson_quadrature(A, r, t, v, sigma, n_gl=48):
    """p = d/dt [ t * M(v t) ] (Eq. 3; spherical mean of Eq. 1) by
    Gauss-Legendre quadrature over mu in [-1, 1], split into pieces dyadic in
    w = 1 - mu so the peak at mu = 1 is resolved.  M'(R) is differentiated
    under the integral sign: p = M(R) + R M'(R), R = v t."""
    R = v * t
    xg, wg = np.polynomial.legendre.leggauss(n_gl)
    a = sigma * sigma / max(R * r, 1e-300) / 4.0
    edges = [0.0]
    e = min(a, 2.0)
    while edges[-1] < 2.0:
        edges.append(min(e, 2.0))
        e *= 2.0
    Msum = 0.0
    Mpsum = 0.0
    for lo, hi in zip(edges[:-1], edges[1:]):
        w = 0.5 * (hi - lo) * xg + 0.5 * (hi + lo)
        wt = 0.5 * (hi - lo) * wg
        mu = 1.0 - w
        expo = -((R - r) ** 2 + 2.0 * R * r * w) / (2.0 * sigma * sigma)
        f = np.exp(expo)
        Msum += np.sum(wt * f)
        Mpsum += np.sum(wt * f * (-(R - r * mu) / (sigma * sigma)))
    M = 0.5 * A * Msum
    Mp = 0.5 * A * Mpsum
    return M + R * Mp


@pytest.mark.parametrize("r_over_sigma", [5, 10, 37.3, 100, 400, 800])
def test_P1_eq6_matches_poisson_quadrature(r_over_sigma):
    """Eq. 6 == quadrature of Poisson's solution, incl.
    the A/(2r) amplitude convention (reading R4)."""
    A = 1.7
    r = r_over_sigma * SIG
    peak = A / (2 * r) * SIG * math.exp(-0.5)
    worst = 0.0
    for d_over_sigma in np.linspace(-2.99, 2.99, 41):
        t = (r - d_over_sigma * SIG) / V
        if t < 0:
            continue
        pq = _poisson_quadrature(A, r, t, V, SIG)
        p6 = oracle.pressure_full(A, r, t, V, SIG)
        worst = max(worst, abs(pq - p6) / peak)
    assert worst <= 1e-12, worst


def test_P2_eq6_initial_condition(golden):
    """Eq. 6 at t = 0 equals the Gaussian source Eq. 1."""
    got = oracle.pressure_full(2.0, 2 * SIG, 0.0, V, SIG)
    assert got == pytest.approx(golden["eq6_t0_A2_r2sigma"], rel=4e-16)
    for r in [0.5 * SIG, 3 * SIG, 7 * SIG]:
        assert oracle.pressure_full(1.0, r, 0.0, V, SIG) == pytest.approx(
            math.exp(-r * r / (2 * SIG * SIG)), rel=4e-16)


def test_P3_far_field_neglect_and_truncation():
    """Eq. 6 - Eq. 7 (incoming term) is negligible for r >> sigma, and
    the oracle's Eq. 7 is exactly zero outside -3 sigma < d < 3 sigma."""
    for r_over in [10, 20, 50]:
        r = r_over * SIG
        peak = 1.0 / (2 * r) * SIG * math.exp(-0.5)
        for d_over in np.linspace(-2.99, 2.99, 13):
            t = (r - d_over * SIG) / V
            full = oracle.pressure_full(1.0, r, t, V, SIG)
            out = oracle.pressure_outgoing(1.0, r, t, V, SIG, 3.0)
            bound = (2 * r / SIG) * math.exp(-(r * r) / (2 * SIG * SIG))  # (r+vt)e^{-(r+vt)^2/2s^2}/s
            assert abs(full - out) <= bound * 10 * peak + 4e-16 * abs(out)
    # r = 20 sigma, vt = r
    r = 20 * SIG
    full = oracle.pressure_full(1.0, r, r / V, V, SIG)
    assert abs(full) / (SIG / (2 * r)) < 1e-100
    # truncation: just inside is nonzero, just outside exactly zero
    r = 200 * SIG
    assert oracle.pressure_outgoing(1.0, r, (r - 2.999 * SIG) / V, V, SIG, 3.0) != 0.0
    assert oracle.pressure_outgoing(1.0, r, (r - 3.001 * SIG) / V, V, SIG, 3.0) == 0.0
    assert oracle.pressure_outgoing(1.0, r, (r + 3.001 * SIG) / V, V, SIG, 3.0) == 0.0


def test_P4_known_value(golden):
    """Eq. 7 at A=1, r=20 mm, sigma=0.1 mm, d=+sigma (hand value)."""
    r = 0.02
    t = (r - SIG) / V
    got = oracle.pressure_outgoing(1.0, r, t, V, SIG, 3.0)
    assert got == pytest.approx(golden["eq7_A1_r20mm_sigma0p1mm_d_plus_sigma"], rel=1e-12)


def test_P5_shape_invariants():
    """Oddness in d, zero crossing at t = r/v, extrema +-(A/2r) sigma e^-1/2,
    1/r decay (P:278 'N-shaped', Eq. 7)."""
    r = 0.03
    for dd in [0.1, 0.5, 1.0, 2.2]:
        p_plus = oracle.pressure_outgoing(1.0, r, (r - dd * SIG) / V, V, SIG, 3.0)
        p_minus = oracle.pressure_outgoing(1.0, r, (r + dd * SIG) / V, V, SIG, 3.0)
        assert p_plus == pytest.approx(-p_minus, rel=1e-9)
    # extremum magnitude at d = sigma
    ts = (r - np.linspace(-3, 3, 60001) * SIG) / V
    vals = np.array([oracle.pressure_outgoing(1.0, r, t, V, SIG, 3.0) for t in ts])
    assert vals.max() == pytest.approx(SIG / (2 * r) * math.exp(-0.5), rel=1e-8)
    assert vals.min() == pytest.approx(-SIG / (2 * r) * math.exp(-0.5), rel=1e-8)
    # sampled trace: sign change brackets t = r/v within one sample; 1/r decay
    fs = 40e6
    c = np.zeros((3, 1), np.float32)
    s1 = np.array([[0.0], [0.0], [-0.02]], np.float32)
    s2 = np.array([[0.0], [0.0], [-0.04]], np.float32)
    y1 = oracle.forward(c, [1.0], s1, sigma=SIG, v=V, fs=fs, n_samples=2048)[0]
    y2 = oracle.forward(c, [1.0], s2, sigma=SIG, v=V, fs=fs, n_samples=2048)[0]
    nz = np.nonzero(y1)[0]
    signs = np.sign(y1[nz])
    flip = nz[np.nonzero(np.diff(signs) < 0)[0][0]]
    t_arr = 0.02 / V
    assert flip / fs <= t_arr + 1e-15 and (flip + 1) / fs >= t_arr - 1e-15
    assert np.abs(y1).max() / np.abs(y2).max() == pytest.approx(2.0, rel=0.01)


def _small_problem(seed, nk=(5, 4, 6), ns=12, nt=None, sigma=SIG, t0=0.0, fs=40e6):
    rng = np.random.default_rng(seed)
    c = inputs.grid_centers(*nk, 1e-4, jitter=0.3, seed=seed)
    s = inputs.hemisphere(ns, 0.012)
    if nt is None:
        nt = int((0.0135 / V - t0) * fs)
    op = dict(sigma=sigma, v=V, fs=fs, n_samples=nt, t0=t0, k=3.0)
    return c, s, op, rng


def test_P6_linearity():
    c, s, op, rng = _small_problem(1)
    M = c.shape[1]
    x1, x2 = rng.random(M), rng.standard_normal(M)
    a, b = 0.7, -1.3
    lhs = oracle.forward(c, a * x1 + b * x2, s, **op)
    rhs = a * oracle.forward(c, x1, s, **op) + b * oracle.forward(c, x2, s, **op)
    assert np.linalg.norm(lhs - rhs) / np.linalg.norm(rhs) <= 1e-12


@pytest.mark.parametrize("seed", range(20))
def test_P7_dot_test(seed):
    """<Ax, d> = <x, A^T d> (P:359, P:389 'rigorously derived'); north_star (c)."""
    if seed % 3 == 0:
        c, s, op = inputs.random_suite_case(seed)[0:3]
    else:
        c, s, op, _ = _small_problem(seed, nk=(3 + seed % 5, 4, 2 + seed % 7), ns=5 + 3 * seed,
                                      t0=(seed % 4) * 1e-6, sigma=SIG * (0.5 + 0.05 * seed))
    rng = np.random.default_rng(seed + 77)
    M, Nd = c.shape[1], s.shape[1]
    x = rng.standard_normal(M)
    d = rng.standard_normal((Nd, op["n_samples"]))
    Ax = oracle.forward(c, x, s, **op)
    ATd = oracle.adjoint(c, d, s, **{k: v for k, v in op.items() if k != "n_samples"})
    lhs, rhs = float(np.sum(Ax * d)), float(np.dot(x, ATd))
    assert abs(lhs - rhs) / (np.linalg.norm(Ax) * np.linalg.norm(d)) <= 1e-10


def _brute_force_matrix(c, s, sigma, v, fs, n_samples, t0, k):
    """Independent brute force: every pair, EVERY sample n in [0, N_t), Eq. 7
    with |d| < k sigma.  Returns A with rows (j, n) and columns i."""
    c64 = c.astype(np.float64)
    s64 = s.astype(np.float64)
    M, Nd = c.shape[1], s.shape[1]
    Amat = np.zeros((Nd * n_samples, M))
    tn = t0 + np.arange(n_samples) / fs
    for j in range(Nd):
        for i in range(M):
            dv = c64[:, i] - s64[:, j]
            r = math.sqrt(dv[0] * dv[0] + dv[1] * dv[1] + dv[2] * dv[2])
            d = r - v * tn
            a = np.where(np.abs(d) < k * sigma, d * np.exp(-d * d / (2 * sigma * sigma)) / (2 * r), 0.0)
            Amat[j * n_samples:(j + 1) * n_samples, i] = a
    return Amat


@pytest.mark.parametrize("seed", [0, 1, 4])
def test_P8_dense_matrix_and_brute_force(seed):
    """A x and A^T d equal the brute-force dense matrix (all samples scanned)."""
    if seed == 4:
        c, s, op = inputs.random_suite_case(seed)
    else:
        c, s, op, _ = _small_problem(seed, nk=(3, 3, 2), ns=6, t0=1e-6 * seed)
    Amat = _brute_force_matrix(c, s, **op)
    rng = np.random.default_rng(seed)
    M, Nd = c.shape[1], s.shape[1]
    x = rng.standard_normal(M)
    d = rng.standard_normal((Nd, op["n_samples"]))
    y = oracle.forward(c, x, s, **op)
    g = oracle.adjoint(c, d, s, **{k: v for k, v in op.items() if k != "n_samples"})
    y_ref = (Amat @ x).reshape(Nd, -1)
    g_ref = Amat.T @ d.ravel()
    assert np.linalg.norm(y - y_ref) <= 1e-12 * np.linalg.norm(y_ref)
    assert np.linalg.norm(g - g_ref) <= 1e-12 * np.linalg.norm(g_ref)
    # columns from unit vectors equal the brute-force columns
    for i in range(min(M, 4)):
        e = np.zeros(M)
        e[i] = 1.0
        col = oracle.forward(c, e, s, **op).ravel()
        assert np.allclose(col, Amat[:, i], rtol=0, atol=1e-14 * np.abs(Amat).max())
    # subset rows / cols are exact rows / cols of the full operator
    rows = np.array([Nd - 1, 0], dtype=np.int32)
    assert np.array_equal(oracle.forward(c, x, s, rows=rows, **op), y[rows])
    cols = np.array([M - 1, 1], dtype=np.int64)
    gs = oracle.adjoint(c, d, s, cols=cols, **{k: v for k, v in op.items() if k != "n_samples"})
    assert np.array_equal(gs, g[cols])


def test_P9_finite_difference_gradient():
    """dL/dz of Eq. 23 (lambda = 0) through NPC (Eq. 19) vs central FD;
    north_star (d)."""
    c = inputs.grid_centers(6, 6, 6, 1e-4)
    s = inputs.hemisphere(8, 0.012)
    op = dict(sigma=SIG, v=V, fs=40e6, n_samples=380, t0=0.0, k=3.0)
    geom = {"centers": c, "sensors": s, "op": op}
    rng = np.random.default_rng(9)
    M = c.shape[1]
    b = oracle.forward(c, rng.random(M), s, **op)
    z = rng.uniform(0.3, 1.0, M)
    hp = ir.Hyper()
    L, gz, _ = ir.loss_and_grad(z, b, geom, hp)
    h = 1e-5
    idx = rng.choice(M, 12, replace=False)
    for i in idx:
        zp, zm = z.copy(), z.copy()
        zp[i] += h
        zm[i] -= h
        Lp = ir.loss_and_grad(zp, b, geom, hp)[0]
        Lm = ir.loss_and_grad(zm, b, geom, hp)[0]
        fd = (Lp - Lm) / (2 * h)
        assert fd == pytest.approx(gz[i], rel=1e-6, abs=1e-9 * np.abs(gz).max())
    # clamp mode gradient is dL/dx itself
    hp_c = ir.Hyper(mode="clamp")
    x = rng.uniform(0.0, 1.0, M)
    _, gx, _ = ir.loss_and_grad(x, b, geom, hp_c)
    i = int(idx[0])
    xp, xm = x.copy(), x.copy()
    xp[i] += h
    xm[i] -= h
    fd = (ir.loss_and_grad(xp, b, geom, hp_c)[0] - ir.loss_and_grad(xm, b, geom, hp_c)[0]) / (2 * h)
    assert fd == pytest.approx(gx[i], rel=1e-6)


def test_P10_adam_step1():
    """Bias-corrected Adam from m = v = 0: dz = -eta g / (|g| + eps_a)."""
    hp = ir.Hyper()
    g = np.array([1e-3, -2.0, 0.0, 5e-9])
    z0 = np.array([0.1, 0.2, 0.3, 0.4])
    z, m, v = ir.adam_update(z0, np.zeros(4), np.zeros(4), g, 0.05, 1, hp)
    expect = z0 - 0.05 * g / (np.abs(g) + hp.adam_eps)
    assert np.allclose(z, expect, rtol=1e-14, atol=1e-17)
    assert np.allclose(m, 0.1 * g) and np.allclose(v, 0.001 * g * g)


def test_P11_cawr(golden):
    """Eq. 24."""
    assert ir.cawr(0, 1e-4, 0.1, 50, 1) == pytest.approx(golden["cawr_t0"], rel=1e-15)
    assert ir.cawr(25, 1e-4, 0.1, 50, 1) == pytest.approx(golden["cawr_t25"], rel=1e-14)
    assert ir.cawr(50, 1e-4, 0.1, 50, 1) == pytest.approx(golden["cawr_t50"], rel=1e-15)
    # printed vs SGDR readings coincide for Tmult = 1, differ for Tmult = 2
    for t in range(0, 300, 7):
        assert ir.cawr(t, 1e-4, 0.1, 50, 1, True) == ir.cawr(t, 1e-4, 0.1, 50, 1, False)
    assert ir.cawr(50, 0.0, 1.0, 50, 2, False) == pytest.approx(1.0)  # restart at T0
    assert ir.cawr(100, 0.0, 1.0, 50, 2, False) == pytest.approx(0.5)  # mid of 2nd period (T=100)
    assert ir.cawr(75, 0.0, 1.0, 50, 2, True) == pytest.approx(0.5 * (1 + math.cos(math.pi * 25 / 100)))


def test_P12_npc(golden):
    """Eq. 18-19."""
    assert ir.npc(np.array([0.0]))[0] == pytest.approx(golden["npc_z0"], rel=1e-15)
    assert ir.npc(np.array([-2.0]))[0] == pytest.approx(4.0, rel=1e-7)
    assert ir.npc_chain(np.array([3.0]), np.array([0.5]))[0] == pytest.approx(3.0 * 2 * (0.5 + 1e-8))


def test_P13_symmetry():
    """One kernel at the centre of axis-aligned sensors at radius R: identical traces."""
    R = 0.0125
    s = np.array([[R, -R, 0, 0, 0, 0], [0, 0, R, -R, 0, 0], [0, 0, 0, 0, R, -R]], np.float32)
    c = np.zeros((3, 1), np.float32)
    y = oracle.forward(c, [2.5], s, sigma=SIG, v=V, fs=40e6, n_samples=400)
    assert np.any(y != 0)
    for j in range(1, 6):
        assert np.array_equal(y[0], y[j])


def test_P14_psf():
    """Single-pass A^T A e_i peaks at or next to kernel i."""
    nk = (7, 7, 7)
    c = inputs.grid_centers(*nk, 1e-4)
    s = inputs.hemisphere(64, 0.012)
    op = dict(sigma=SIG, v=V, fs=40e6, n_samples=380, t0=0.0, k=3.0)
    M = c.shape[1]
    for i in [0, M // 2, 3 + 7 * (2 + 7 * 4)]:
        e = np.zeros(M)
        e[i] = 1.0
        y = oracle.forward(c, e, s, **op)
        g = oracle.adjoint(c, y, s, **{k: v for k, v in op.items() if k != "n_samples"})
        j = int(np.argmax(g))
        dist = np.abs(c[:, i].astype(np.float64) - c[:, j]).max()
        assert dist <= 1.01e-4


def test_geometry_error_when_sensor_inside_kernel_support():
    c = np.zeros((3, 1), np.float32)
    s = np.array([[2e-4], [0.0], [0.0]], np.float32)  # r = 2 sigma < 3 sigma
    with pytest.raises(oracle.OracleGeometryError):
        oracle.forward(c, [1.0], s, sigma=SIG, v=V, fs=40e6, n_samples=10)


def test_thread_count_invariance():
    c, s, op, rng = _small_problem(5)
    x = rng.random(c.shape[1])
    oracle.set_threads(1)
    y1 = oracle.forward(c, x, s, **op)
    oracle.set_threads(4)
    y4 = oracle.forward(c, x, s, **op)
    oracle.set_threads(0)
    assert np.array_equal(y1, y4)


def test_pair_sample_count_matches_brute_force():
    c, s, op, _ = _small_problem(2, nk=(3, 3, 3), ns=7)
    Amat = _brute_force_matrix(c, s, **op)
    assert oracle.count_pair_samples(c, s, **op) == int(np.count_nonzero(Amat))


def test_forward_trace_equals_pinned_eq7():
    """The forward's per-pair entries equal the scalar Eq. 7 (pinned above by
    the quadrature P1/P3 and the hand value P4) at every sample t_n = t0 + n/f_s."""
    c = np.array([[1e-4], [-2e-4], [3e-4]], np.float32)
    s = np.array([[0.004], [-0.009], [-0.011]], np.float32)
    fs, t0 = 40e6, 1.5e-6
    y = oracle.forward(c, [1.7], s, sigma=SIG, v=V, fs=fs, n_samples=600, t0=t0)[0]
    r = float(np.sqrt(np.sum((c[:, 0].astype(np.float64) - s[:, 0]) ** 2)))
    ref = np.array([1.7 * oracle.pressure_outgoing(1.0, r, t0 + n / fs, V, SIG, 3.0) for n in range(600)])
    assert np.count_nonzero(ref) >= 15
    assert np.allclose(y, ref, rtol=1e-14, atol=0)
