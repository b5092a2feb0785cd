"""Vessel continuity regularisation (Eqs. 20-22,
P:457-481) in plain numpy fp64 -- TEST INFRASTRUCTURE ONLY.

    R_VCR(x) = R_H(x) + beta R_TV(x)                                  (Eq. 20)
    R_H(x)   = sum_i sqrt( sum_{p,q in {x,y,z}} (D_pq x_i)^2 + eps )   (Eq. 21)
    R_TV(x)  = sum_i sqrt( sum_{d in {x,y,z}} (D_d x_i)^2 + eps )      (Eq. 22)

on the voxel grid with i = ix + nx (iy + ny iz) (the order of the kernel
centres).  The paper names the operators only; readings V1-V4 of
DESIGN.md fix them:
  V1 D_d: forward difference x(i + e_d) - x(i), 0 at the last index (replicate
     boundary).
  V2 D_pp: [1, -2, 1] on the nearest interior stencil, centre clamp(i, 1, n-2)
     (0 if n < 3), so affine images have zero second differences everywhere.
  V3 D_pq (p != q): forward-forward cross difference x(i+e_p+e_q) - x(i+e_p)
     - x(i+e_q) + x(i) with replicate clamping (0 on the last index of p or q);
     both orderings pq and qp are summed, i.e. mixed terms count twice.
  V4 eps: independent of the NPC epsilon (reading R16), default 1e-8.
The gradient is the exact adjoint of each difference operator applied to
w_i D x_i / s_i, written out per stencil (no autodiff).
"""
from __future__ import annotations

import numpy as np


def _grid(x, dims):
    nx, ny, nz = dims
    return np.asarray(x, dtype=np.float64).reshape(nz, ny, nx)  # [iz, iy, ix]


def _shift(a, axis, step):
    """a(i + step e_axis) with replicate clamping."""
    n = a.shape[axis]
    idx = np.clip(np.arange(n) + step, 0, n - 1)
    return np.take(a, idx, axis=axis)


def _fwd(a, axis):
    """V1: forward difference with replicate boundary."""
    return _shift(a, axis, 1) - a


def _fwd_T(u, axis):
    """Adjoint of _fwd: (D^T u)(k) = u(k-1)[k-1 valid, not last] - u(k)[k not last]."""
    n = u.shape[axis]
    v = u.copy()
    last = [slice(None)] * u.ndim
    last[axis] = n - 1
    v[tuple(last)] = 0.0  # D is 0 at the last index, whatever u is there
    g = -v
    prev = [slice(None)] * u.ndim
    prev[axis] = slice(1, None)
    src = [slice(None)] * u.ndim
    src[axis] = slice(0, n - 1)
    g[tuple(prev)] += v[tuple(src)]
    return g


def _second(a, axis):
    """V2: [1,-2,1] on the nearest interior stencil."""
    n = a.shape[axis]
    if n < 3:
        return np.zeros_like(a)
    c = np.clip(np.arange(n), 1, n - 2)
    return np.take(a, c + 1, axis=axis) - 2.0 * np.take(a, c, axis=axis) + np.take(a, c - 1, axis=axis)


def _second_T(u, axis):
    n = u.shape[axis]
    g = np.zeros_like(u)
    if n < 3:
        return g
    c = np.clip(np.arange(n), 1, n - 2)
    for i in range(n):
        ui = np.take(u, i, axis=axis)
        for off, w in ((1, 1.0), (0, -2.0), (-1, 1.0)):
            sl = [slice(None)] * u.ndim
            sl[axis] = c[i] + off
            g[tuple(sl)] += w * ui
    return g


def _mixed(a, p, q):
    """V3: forward-forward cross difference with replicate clamping."""
    return _shift(_shift(a, p, 1), q, 1) - _shift(a, p, 1) - _shift(a, q, 1) + a


def _mixed_T(u, p, q):
    """Adjoint of _mixed, by explicit index bookkeeping of the 4 taps."""
    g = np.zeros_like(u)
    shape = u.shape
    idx = np.indices(shape)
    taps = (((1, 1), 1.0), ((1, 0), -1.0), ((0, 1), -1.0), ((0, 0), 1.0))
    for (sp, sq), w in taps:
        tgt = [ix.copy() for ix in idx]
        tgt[p] = np.minimum(tgt[p] + sp, shape[p] - 1)
        tgt[q] = np.minimum(tgt[q] + sq, shape[q] - 1)
        np.add.at(g, tuple(tgt), w * u)
    return g


AXES = {"x": 2, "y": 1, "z": 0}


def hessian_terms(a):
    """List of (D_pq a, multiplicity) over the 6 distinct stencils."""
    out = []
    for d in "xyz":
        out.append((("pp", AXES[d]), 1.0))
    for p, q in (("x", "y"), ("x", "z"), ("y", "z")):
        out.append((("pq", AXES[p], AXES[q]), 2.0))
    return out


def _apply(a, op):
    return _second(a, op[1]) if op[0] == "pp" else _mixed(a, op[1], op[2])


def _apply_T(u, op):
    return _second_T(u, op[1]) if op[0] == "pp" else _mixed_T(u, op[1], op[2])


def r_tv(x, dims, eps=1e-8, grad=True):
    """Eq. 22 value and gradient."""
    a = _grid(x, dims)
    D = [_fwd(a, ax) for ax in (2, 1, 0)]
    s = np.sqrt(sum(d * d for d in D) + eps)
    val = float(s.sum())
    if not grad:
        return val
    g = sum(_fwd_T(d / s, ax) for d, ax in zip(D, (2, 1, 0)))
    return val, g.ravel()


def r_hessian(x, dims, eps=1e-8, grad=True):
    """Eq. 21 value and gradient (Frobenius form, mixed terms twice)."""
    a = _grid(x, dims)
    terms = [(op, mult, _apply(a, op)) for op, mult in hessian_terms(a)]
    s = np.sqrt(sum(mult * d * d for _, mult, d in terms) + eps)
    val = float(s.sum())
    if not grad:
        return val
    g = sum(mult * _apply_T(d / s, op) for op, mult, d in terms)
    return val, g.ravel()


def r_vcr(x, dims, beta, eps=1e-8):
    """Eq. 20: R_H + beta R_TV, value and gradient."""
    vh, gh = r_hessian(x, dims, eps)
    vt, gt = r_tv(x, dims, eps)
    return vh + beta * vt, gh + beta * gt
