"""fp64 CPU oracle for the GPAIR hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product package ``paper_2602_03893_b200`` never imports it, and it never
imports the product package: the two share no code.  Seeded inputs come from
``gpair_inputs`` (a module with none of the method's arithmetic) and are
passed in by the caller.

Contents
--------
* ``forward`` / ``adjoint``: ctypes wrappers over ``gpair_oracle.c`` -- the
  direct enumeration of Eq. 7 in fp64.
* ``pressure_full`` / ``pressure_outgoing``: Eq. 6 and Eq. 7 with
  the P:291 truncation, scalar fp64.
* ``ir``: Algorithm 2 -- NPC, loss, chain rule, CAWR, Adam -- in
  plain numpy fp64 (see ``oracle/ir.py``).

Parity status: every function here is pinned by ``tests/test_oracle_pins.py``
(quadrature of Poisson's formula, closed-form values, dot test, dense matrix,
brute force, finite differences).  Nothing is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gpair_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

CFLAGS = ["-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile the oracle shared library (gcc, fp64, no fast-math)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _LIB_PATH, _SRC, "-lm"])
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        d, i32, i64 = ctypes.c_double, ctypes.c_int32, ctypes.c_int64
        vp = ctypes.c_void_p
        L.oracle_pressure_full.restype = d
        L.oracle_pressure_full.argtypes = [d, d, d, d, d]
        L.oracle_pressure_outgoing.restype = d
        L.oracle_pressure_outgoing.argtypes = [d, d, d, d, d, d]
        L.oracle_forward.restype = ctypes.c_int
        L.oracle_forward.argtypes = [i64, vp, vp, d, vp, i32, vp, d, d, d, i32, d, vp, i32, vp]
        L.oracle_adjoint.restype = ctypes.c_int
        L.oracle_adjoint.argtypes = [i64, vp, d, vp, i32, vp, d, d, d, i32, d, vp, vp, i64, vp]
        L.oracle_forward_nf.restype = ctypes.c_int
        L.oracle_forward_nf.argtypes = L.oracle_forward.argtypes
        L.oracle_adjoint_nf.restype = ctypes.c_int
        L.oracle_adjoint_nf.argtypes = L.oracle_adjoint.argtypes
        L.oracle_count_pair_samples.restype = i64
        L.oracle_count_pair_samples.argtypes = [i64, vp, d, i32, vp, d, d, d, i32, d, vp, i64]
        L.oracle_assa_taps.restype = None
        L.oracle_assa_taps.argtypes = [d, d, d, i32, d, vp]
        L.oracle_assa_forward.restype = ctypes.c_int
        L.oracle_assa_forward.argtypes = [i64, vp, vp, i32, vp, d, d, d, i32, d, d, i32, i32, vp, i32, vp]
        L.oracle_assa_adjoint.restype = ctypes.c_int
        L.oracle_assa_adjoint.argtypes = [i64, vp, i32, vp, d, d, d, i32, d, d, i32, i32, vp, vp, i64, vp]
        L.oracle_set_threads.argtypes = [ctypes.c_int]
        L.oracle_get_threads.restype = ctypes.c_int
        _lib = L
    return _lib


class OracleGeometryError(ValueError):
    pass


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f32_soa(a, n):
    a = np.ascontiguousarray(a, dtype=np.float32)
    if a.shape != (3, n):
        raise ValueError(f"expected SoA [3][{n}] float32, got {a.shape}")
    return a


def set_threads(n: int) -> None:
    lib().oracle_set_threads(int(n))


def threads() -> int:
    return int(lib().oracle_get_threads())


def pressure_full(A, r, t, v, sigma):
    """Eq. 6, fp64 scalar."""
    return lib().oracle_pressure_full(A, r, t, v, sigma)


def pressure_outgoing(A, r, t, v, sigma, k=3.0):
    """Eq. 7 truncated to |d| < k sigma, fp64 scalar."""
    return lib().oracle_pressure_outgoing(A, r, t, v, sigma, k)


def forward(centers, amp, sensors, *, sigma, v, fs, n_samples, t0=0.0, k=3.0,
            sigmas=None, rows=None, near_field=False):
    """y = A x by direct enumeration. Returns fp64 [n_rows][N_t].

    centers: [3][M] float32 SoA (metres); amp: [M] (promoted to fp64);
    sensors: [3][N_d] float32 SoA; rows: optional sensor subset (exact rows);
    sigmas: optional per-kernel sigma_i [M] (row f4, reading N2);
    near_field: Eq. 6 with both terms (row f4, reading N1), pairs need r > 0.
    """
    amp = np.ascontiguousarray(amp, dtype=np.float64)
    M = amp.shape[0]
    c = _f32_soa(centers, M)
    Nd = np.asarray(sensors).shape[1]
    s = _f32_soa(sensors, Nd)
    sg = None if sigmas is None else np.ascontiguousarray(sigmas, dtype=np.float64)
    if rows is not None:
        rows = np.ascontiguousarray(rows, dtype=np.int32)
        n_rows = rows.shape[0]
    else:
        n_rows = Nd
    y = np.zeros((n_rows, int(n_samples)), dtype=np.float64)
    fn = lib().oracle_forward_nf if near_field else lib().oracle_forward
    rc = fn(M, _ptr(c), _ptr(amp), float(sigma), _ptr(sg), Nd, _ptr(s),
            float(v), float(fs), float(t0), int(n_samples), float(k), _ptr(rows), n_rows, _ptr(y))
    if rc == 2:
        raise OracleGeometryError("r_ij = 0" if near_field else
                                  "a kernel-sensor distance r_ij <= k*sigma (far-field model invalid)")
    if rc != 0:
        raise ValueError(f"oracle_forward: invalid argument (rc={rc})")
    return y


def adjoint(centers, delta, sensors, *, sigma, v, fs, t0=0.0, k=3.0, sigmas=None, cols=None,
            n_kernels=None, near_field=False):
    """g = A^T delta (exact transpose of ``forward``). Returns fp64 [n_cols]."""
    delta = np.ascontiguousarray(delta, dtype=np.float64)
    Nd, Nt = delta.shape
    M = int(n_kernels) if n_kernels is not None else np.asarray(centers).shape[1]
    c = _f32_soa(centers, M)
    s = _f32_soa(sensors, Nd)
    sg = None if sigmas is None else np.ascontiguousarray(sigmas, dtype=np.float64)
    if cols is not None:
        cols = np.ascontiguousarray(cols, dtype=np.int64)
        n_cols = cols.shape[0]
    else:
        n_cols = M
    g = np.zeros(n_cols, dtype=np.float64)
    fn = lib().oracle_adjoint_nf if near_field else lib().oracle_adjoint
    rc = fn(M, _ptr(c), float(sigma), _ptr(sg), Nd, _ptr(s), float(v), float(fs),
            float(t0), Nt, float(k), _ptr(delta), _ptr(cols), n_cols, _ptr(g))
    if rc == 2:
        raise OracleGeometryError("r_ij = 0" if near_field else
                                  "a kernel-sensor distance r_ij <= k*sigma (far-field model invalid)")
    if rc != 0:
        raise ValueError(f"oracle_adjoint: invalid argument (rc={rc})")
    return g


def count_pair_samples(centers, sensors, *, sigma, v, fs, n_samples, t0=0.0, k=3.0, cols=None):
    """Exact number of in-window (n in [0,N_t)) pair-samples of the operator."""
    c = np.ascontiguousarray(centers, dtype=np.float32)
    M = c.shape[1]
    s = np.ascontiguousarray(sensors, dtype=np.float32)
    Nd = s.shape[1]
    if cols is not None:
        cols = np.ascontiguousarray(cols, dtype=np.int64)
        n_cols = cols.shape[0]
    else:
        n_cols = M
    return int(lib().oracle_count_pair_samples(M, _ptr(c), float(sigma), Nd, _ptr(s), float(v),
                                               float(fs), float(t0), int(n_samples), float(k),
                                               _ptr(cols), n_cols))


# ---------------------------------------------------------------- ASSA (row f1)
def assa_params(sigma, v, fs, k=3.0, n_min=25):
    """Eq. 8.  N_half = ceil(k sigma / (v dt)) -- the ratio is
    rounded to 12 significant digits before the ceiling so that an exact
    integer ratio (8.0 at sigma = 0.1 mm, f_s = 40 MHz) is not pushed up by
    its binary representation (reading A2); alpha = max(1, ceil(((N_min-1)/2)
    / N_half)) in exact integer arithmetic; K = alpha N_half."""
    ratio = float(f"{k * sigma * fs / v:.12g}")
    n_half = max(1, int(math.ceil(ratio)))
    num, den = n_min - 1, 2 * n_half  # ceil((N_min - 1) / (2 N_half))
    alpha = max(1, -(-num // den))
    return {"n_half": n_half, "alpha": alpha, "K": alpha * n_half, "fs_up": alpha * fs, "n_min": n_min}


def assa_taps(sigma, v, fs_up, K, C=0.5):
    """Eq. 11, h[k + K] for k = -K..K."""
    h = np.zeros(2 * K + 1)
    lib().oracle_assa_taps(float(v), float(fs_up), float(sigma), int(K), float(C), _ptr(h))
    return h


def assa_forward(centers, amp, sensors, *, sigma, v, fs, n_samples, alpha, K, t0=0.0, k=3.0, rows=None):
    """ASSA forward y = S_down(h * P_up x) (Eq. 13), Algorithm 1 ForwardOp."""
    amp = np.ascontiguousarray(amp, dtype=np.float64)
    M = amp.shape[0]
    c = _f32_soa(centers, M)
    Nd = np.asarray(sensors).shape[1]
    s = _f32_soa(sensors, Nd)
    if rows is not None:
        rows = np.ascontiguousarray(rows, dtype=np.int32)
        n_rows = rows.shape[0]
    else:
        n_rows = Nd
    y = np.zeros((n_rows, int(n_samples)), dtype=np.float64)
    rc = lib().oracle_assa_forward(M, _ptr(c), _ptr(amp), Nd, _ptr(s), float(v), float(fs), float(t0),
                                   int(n_samples), float(sigma), float(k), int(alpha), int(K), _ptr(rows), n_rows,
                                   _ptr(y))
    if rc == 2:
        raise OracleGeometryError("a kernel-sensor distance r_ij <= k*sigma")
    if rc != 0:
        raise ValueError(f"oracle_assa_forward: invalid argument (rc={rc})")
    return y


def assa_adjoint(centers, delta, sensors, *, sigma, v, fs, alpha, K, t0=0.0, k=3.0, cols=None, n_kernels=None):
    """ASSA adjoint g = P_up^T (h-bar * S_down^T delta) (Eq. 14), Algorithm 1 AdjointOp."""
    delta = np.ascontiguousarray(delta, dtype=np.float64)
    Nd, Nt = delta.shape
    M = int(n_kernels) if n_kernels is not None else np.asarray(centers).shape[1]
    c = _f32_soa(centers, M)
    s = _f32_soa(sensors, Nd)
    if cols is not None:
        cols = np.ascontiguousarray(cols, dtype=np.int64)
        n_cols = cols.shape[0]
    else:
        n_cols = M
    g = np.zeros(n_cols, dtype=np.float64)
    rc = lib().oracle_assa_adjoint(M, _ptr(c), Nd, _ptr(s), float(v), float(fs), float(t0), Nt, float(sigma),
                                   float(k), int(alpha), int(K), _ptr(delta), _ptr(cols), n_cols, _ptr(g))
    if rc == 2:
        raise OracleGeometryError("a kernel-sensor distance r_ij <= k*sigma")
    if rc != 0:
        raise ValueError(f"oracle_assa_adjoint: invalid argument (rc={rc})")
    return g
