"""Pins of the VCR oracle (row f2; Eqs. 20-22):
closed-form values (constant and affine images, single voxel), exact
invariances (translation, homogeneity of the smoothed form), and central
finite differences of the value for the gradient."""
import math

import numpy as np
import pytest

from oracle import vcr


@pytest.mark.parametrize("dims", [(4, 4, 4), (5, 3, 2), (1, 1, 1), (2, 7, 3)])
def test_constant_image(dims):
    M = int(np.prod(dims))
    x = np.full(M, 3.25)
    for eps in (1e-8, 1e-3):
        assert vcr.r_tv(x, dims, eps, grad=False) == pytest.approx(M * math.sqrt(eps), rel=1e-14)
        assert vcr.r_hessian(x, dims, eps, grad=False) == pytest.approx(M * math.sqrt(eps), rel=1e-14)
        v, g = vcr.r_vcr(x, dims, 1.0, eps)
        assert v == pytest.approx(2 * M * math.sqrt(eps), rel=1e-14)
        assert np.abs(g).max() <= 1e-12


def test_affine_image_has_zero_hessian():
    dims = (6, 5, 4)
    iz, iy, ix = np.meshgrid(*(np.arange(n) for n in dims[::-1]), indexing="ij")
    x = (0.3 + 0.7 * ix - 1.1 * iy + 0.25 * iz).ravel()
    M = x.size
    v, g = vcr.r_hessian(x, dims, 1e-6)
    assert v == pytest.approx(M * math.sqrt(1e-6), rel=1e-12)
    assert np.abs(g).max() <= 1e-9
    # TV of the same ramp: sqrt(b.b + eps) on the interior faces
    assert vcr.r_tv(x, dims, 1e-6, grad=False) > M * math.sqrt(1e-6)


def test_translation_and_homogeneity():
    rng = np.random.default_rng(0)
    dims = (5, 4, 3)
    x = rng.standard_normal(int(np.prod(dims)))
    for f in (vcr.r_tv, vcr.r_hessian):
        assert f(x + 7.0, dims, 1e-8, grad=False) == pytest.approx(f(x, dims, 1e-8, grad=False), rel=1e-12)
        c = 2.5  # R(c x; c^2 eps) = c R(x; eps)
        assert f(c * x, dims, c * c * 1e-4, grad=False) == pytest.approx(c * f(x, dims, 1e-4, grad=False), rel=1e-12)


@pytest.mark.parametrize("dims", [(4, 4, 4), (5, 3, 2), (3, 1, 6)])
@pytest.mark.parametrize("which", ["tv", "h", "vcr"])
def test_gradient_vs_finite_differences(dims, which):
    rng = np.random.default_rng(hash((dims, which)) % 2**32)
    M = int(np.prod(dims))
    x = rng.uniform(0.0, 1.0, M)
    eps = 1e-3
    if which == "tv":
        f = lambda z: vcr.r_tv(z, dims, eps)  # noqa: E731
    elif which == "h":
        f = lambda z: vcr.r_hessian(z, dims, eps)  # noqa: E731
    else:
        f = lambda z: vcr.r_vcr(z, dims, 0.7, eps)  # noqa: E731
    _, g = f(x)
    h = 1e-6
    for i in range(M):
        xp, xm = x.copy(), x.copy()
        xp[i] += h
        xm[i] -= h
        fd = (f(xp)[0] - f(xm)[0]) / (2 * h)
        assert fd == pytest.approx(g[i], rel=1e-6, abs=1e-7)


def test_stencils_by_hand():
    """Single nonzero voxel at the interior: the second differences and mixed
    differences around it have the textbook values."""
    dims = (5, 5, 5)
    a = np.zeros(dims[::-1])
    a[2, 2, 2] = 1.0
    assert vcr._second(a, 2)[2, 2, 2] == -2.0 and vcr._second(a, 2)[2, 2, 1] == 1.0
    m = vcr._mixed(a, 2, 1)  # D_xy: x(i+ex+ey) - x(i+ex) - x(i+ey) + x(i)
    assert m[2, 2, 2] == 1.0 and m[2, 1, 1] == 1.0 and m[2, 1, 2] == -1.0 and m[2, 2, 1] == -1.0


def test_ir_gradient_with_vcr_vs_finite_differences():
    """Eq. 23 with lambda > 0: dL/dz through NPC matches central FD."""
    import oracle
    from oracle import ir
    from paper_2602_03893_b200 import inputs

    dims = (4, 4, 3)
    c = inputs.grid_centers(*dims, 1e-4)
    s = inputs.hemisphere(6, 0.012)
    op = dict(sigma=1e-4, v=1500.0, fs=40e6, n_samples=380, t0=0.0, k=3.0)
    geom = {"centers": c, "sensors": s, "op": op}
    rng = np.random.default_rng(2)
    M = c.shape[1]
    b = oracle.forward(c, rng.random(M), s, **op)
    z = rng.uniform(0.3, 1.0, M)
    hp = ir.Hyper(lam=3e-3, beta=0.5, eps_reg=1e-4, dims=dims)
    _, gz, _ = ir.loss_and_grad(z, b, geom, hp)
    h = 1e-5
    for i in rng.choice(M, 8, replace=False):
        zp, zm = z.copy(), z.copy()
        zp[i] += h
        zm[i] -= h
        fd = (ir.loss_and_grad(zp, b, geom, hp)[0] - ir.loss_and_grad(zm, b, geom, hp)[0]) / (2 * h)
        assert fd == pytest.approx(gz[i], rel=1e-6, abs=1e-9 * np.abs(gz).max())


@pytest.mark.parametrize("z0,z1", [(0, 4), (3, 6), (5, 9), (9, 14), (12, 14)])
def test_gradient_halo_is_two_planes(z0, z1):
    """Kernel sharding of R_VCR (z-slab halo exchange,
    2 planes): the gradient on the z planes [z0, z1) of the
    whole-grid R_VCR depends on x only through the planes [z0-2, z1+2), so a
    2-plane halo per side is enough and a 1-plane halo is not.  Pinned on the
    oracle alone: perturbing every plane outside the halo leaves the own-plane
    gradient bit-identical, perturbing plane z0-2 (or z1+1) changes it."""
    dims = (5, 4, 14)
    nx, ny, nz = dims
    rng = np.random.default_rng(100 + z0)
    a = rng.uniform(0.0, 1.0, (nz, ny, nx))
    own = slice(z0 * nx * ny, z1 * nx * ny)
    _, g = vcr.r_vcr(a.ravel(), dims, 0.7, 1e-3)
    b = a.copy()
    lo, hi = max(0, z0 - 2), min(nz, z1 + 2)
    b[:lo] = rng.uniform(0.0, 1.0, b[:lo].shape)
    b[hi:] = rng.uniform(0.0, 1.0, b[hi:].shape)
    _, gb = vcr.r_vcr(b.ravel(), dims, 0.7, 1e-3)
    assert np.array_equal(g[own], gb[own])
    for p in (z0 - 2, z1 + 1):
        if 0 <= p < nz and not (z0 <= p < z1):
            c = a.copy()
            c[p] += 0.5
            _, gc = vcr.r_vcr(c.ravel(), dims, 0.7, 1e-3)
            assert np.abs(gc[own] - g[own]).max() > 1e-6, p
