"""Seeded synthetic inputs shaped like the paper's workloads.

This module holds NONE of the method's arithmetic (no distances, windows,
exponentials or operator entries): it only builds kernel grids, sensor arrays,
amplitudes and residuals.  It is the one module both the oracle-side tests and
the CUDA-side harness use, so both operate on identical inputs.  The recipe is
SURVEY.md section 8(d) and DESIGN.md section "Input recipe":

* kernel centres on a grid centred on the origin, index i = ix + nx (iy + ny iz)
  (SPEC S:27), spacing dx, sigma = dx;
* hemispherical array: lower half, Fibonacci placement,
  radius 60 mm;
* planar array: checkerboard half of a 32x32 lattice at 3.2 mm pitch
  (102.4 mm aperture), 5 mm below the volume (limited view, sparse);
* amplitudes: dense U[0,1) (throughput input), vessel phantom (random-walk
  tubes, mirrors the paper's vascular ground truth P:67), single kernel;
* residual for adjoint parity: N(0,1).

All positions are float32 metres in SoA layout [3][n].
"""
from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np

MM = 1e-3


def grid_centers(nx, ny, nz, dx, jitter=0.0, seed=0):
    """Kernel centres c_i = o + dx (ix, iy, iz), o centring the grid on 0.

    Returns float32 [3][nx*ny*nz] with i = ix + nx (iy + ny iz).
    ``jitter`` (fraction of dx) adds U[-j, j] dx per coordinate (random suite).
    """
    ix = np.arange(nx, dtype=np.float64) - (nx - 1) / 2.0
    iy = np.arange(ny, dtype=np.float64) - (ny - 1) / 2.0
    iz = np.arange(nz, dtype=np.float64) - (nz - 1) / 2.0
    Z, Y, X = np.meshgrid(iz, iy, ix, indexing="ij")
    c = np.stack([X.ravel(), Y.ravel(), Z.ravel()]) * dx
    if jitter:
        rng = np.random.default_rng(seed)
        c = c + rng.uniform(-jitter, jitter, size=c.shape) * dx
    return np.ascontiguousarray(c.astype(np.float32))


def hemisphere(n, radius, center=(0.0, 0.0, 0.0)):
    """Lower-hemisphere Fibonacci array: mu_j = -(j+0.5)/n."""
    j = np.arange(n, dtype=np.float64)
    mu = -(j + 0.5) / n
    rho = np.sqrt(1.0 - mu * mu)
    phi = j * math.pi * (3.0 - math.sqrt(5.0))
    s = np.stack([rho * np.cos(phi), rho * np.sin(phi), mu]) * radius
    s += np.asarray(center, dtype=np.float64)[:, None]
    return np.ascontiguousarray(s.astype(np.float32))


def planar_checkerboard(n_side=32, pitch=3.2 * MM, z=-11.4 * MM, parity=0):
    """Config-5 sparse limited-view planar array: (ix+iy) even half of a lattice."""
    pts = []
    for iy in range(n_side):
        for ix in range(n_side):
            if (ix + iy) % 2 == parity:
                pts.append(((ix - (n_side - 1) / 2.0) * pitch, (iy - (n_side - 1) / 2.0) * pitch, z))
    return np.ascontiguousarray(np.asarray(pts, dtype=np.float64).T.astype(np.float32))


def dense_amplitudes(M, seed=1):
    """Throughput input: U[0,1) (work does not depend on values)."""
    return np.random.default_rng(seed).random(M).astype(np.float32)


def residual(n_sensors, n_samples, seed=3):
    """Adjoint parity input: N(0,1) residual [N_d][N_t]."""
    return np.random.default_rng(seed).standard_normal((n_sensors, n_samples)).astype(np.float32)


def vessel_phantom(nx, ny, nz, seed=2, n_tubes=None):
    """Random-walk tubes on the voxel grid (SURVEY 8d amplitude (ii)).

    max(4, M/65536) tubes of 12 segments, each 8 voxels long with turns of at
    most 30 degrees, radius U[1,3] voxels; amplitude exp(-dist^2 / (2 rho^2))
    (max over segments), zeroed below 1e-3.  Units: voxel indices.
    """
    M = nx * ny * nz
    rng = np.random.default_rng(seed)
    n_tubes = n_tubes or max(4, M // 65536)
    amp = np.zeros((nz, ny, nx), dtype=np.float64)
    dims = np.array([nx, ny, nz], dtype=np.float64)
    for _ in range(n_tubes):
        p = rng.uniform(0.2, 0.8, 3) * (dims - 1)
        d = rng.standard_normal(3)
        d /= np.linalg.norm(d)
        rad = rng.uniform(1.0, 3.0)
        for _s in range(12):
            # turn by at most 30 degrees
            while True:
                q = rng.standard_normal(3)
                q -= q.dot(d) * d
                nq = np.linalg.norm(q)
                if nq > 1e-9:
                    break
            q /= nq
            ang = math.radians(rng.uniform(0.0, 30.0))
            d = math.cos(ang) * d + math.sin(ang) * q
            p1 = p + 8.0 * d
            reach = int(math.ceil(rad * 3.8)) + 1
            lo = np.maximum(np.floor(np.minimum(p, p1)) - reach, 0).astype(int)
            hi = np.minimum(np.ceil(np.maximum(p, p1)) + reach, dims - 1).astype(int)
            if np.all(hi >= lo):
                zz, yy, xx = np.meshgrid(np.arange(lo[2], hi[2] + 1), np.arange(lo[1], hi[1] + 1),
                                         np.arange(lo[0], hi[0] + 1), indexing="ij")
                pts = np.stack([xx, yy, zz], axis=-1).astype(np.float64)
                seg = p1 - p
                tt = np.clip(((pts - p) @ seg) / seg.dot(seg), 0.0, 1.0)
                near = p + tt[..., None] * seg
                dist2 = np.sum((pts - near) ** 2, axis=-1)
                val = np.exp(-dist2 / (2.0 * rad * rad))
                sub = amp[lo[2]:hi[2] + 1, lo[1]:hi[1] + 1, lo[0]:hi[0] + 1]
                np.maximum(sub, val, out=sub)
            p = np.clip(p1, 0, dims - 1)
    amp[amp < 1e-3] = 0.0
    return amp.ravel().astype(np.float32)


def blobs_phantom(nx, ny, nz, count=5, seed=5):
    """Desk-scale phantom ("blobs"): `count`
    isotropic Gaussian blobs, centres U[0.25, 0.75] of each axis, std-dev
    U[1.5, 3] voxels, peak U[0.5, 1]; max over blobs, zeroed below 1e-3.
    Units: voxel indices; returns float32 [M] in grid order."""
    rng = np.random.default_rng(seed)
    zz, yy, xx = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    amp = np.zeros((nz, ny, nx), dtype=np.float64)
    dims = np.array([nx, ny, nz], dtype=np.float64)
    for _ in range(count):
        c = rng.uniform(0.25, 0.75, 3) * (dims - 1)
        rad = rng.uniform(1.5, 3.0)
        peak = rng.uniform(0.5, 1.0)
        d2 = (xx - c[0]) ** 2 + (yy - c[1]) ** 2 + (zz - c[2]) ** 2
        np.maximum(amp, peak * np.exp(-d2 / (2.0 * rad * rad)), out=amp)
    amp[amp < 1e-3] = 0.0
    return amp.ravel().astype(np.float32)


def add_noise(b, snr, seed=9):
    """Additive zero-mean Gaussian noise with max|b| / std = snr (SPEC S:708,
    the amplitude reading of the paper's "SNR ~ 5:1")."""
    rng = np.random.default_rng(seed)
    std = float(np.abs(b).max()) / snr
    return (b + rng.standard_normal(b.shape) * std).astype(b.dtype)


@dataclass(frozen=True)
class Config:
    """One workload of SURVEY.md section 8(d) (BASELINE.json configs)."""
    name: str
    grid: tuple  # (nx, ny, nz)
    dx: float  # kernel spacing [m]
    array: str  # "hemisphere" | "planar"
    n_sensors: int
    radius: float  # hemisphere radius [m]
    n_samples: int
    fs: float = 40e6  # sampling rate [Hz] (proposed)
    v: float = 1500.0  # speed of sound [m/s]
    sigma: float | None = None  # None -> dx
    k: float = 3.0  # truncation
    t0: float = 0.0

    @property
    def M(self):
        return self.grid[0] * self.grid[1] * self.grid[2]

    @property
    def sig(self):
        return self.dx if self.sigma is None else self.sigma

    def centers(self):
        return grid_centers(*self.grid, self.dx)

    def sensors(self):
        if self.array == "hemisphere":
            return hemisphere(self.n_sensors, self.radius)
        s = planar_checkerboard()
        assert s.shape[1] == self.n_sensors
        return s

    def op_kwargs(self):
        return dict(sigma=self.sig, v=self.v, fs=self.fs, n_samples=self.n_samples, t0=self.t0, k=self.k)


CONFIGS = {
    "cfg1": Config("cfg1", (8, 8, 8), 0.1 * MM, "hemisphere", 64, 12.8 * MM, 512),
    "cfg2": Config("cfg2", (64, 64, 64), 0.1 * MM, "hemisphere", 256, 60 * MM, 2048),
    "cfg3": Config("cfg3", (128, 128, 128), 0.1 * MM, "hemisphere", 1024, 60 * MM, 4096),
    "cfg4": Config("cfg4", (256, 256, 128), 0.1 * MM, "hemisphere", 1024, 60 * MM, 4096),
    "cfg5": Config("cfg5", (256, 256, 128), 0.1 * MM, "planar", 512, 0.0, 4096),
    # desk-scale reconstruction workload (row f3): 32^3 at 0.4 mm,
    # 64-element hemisphere of radius 25 mm, W = 64 samples per pair
    "desk": Config("desk", (32, 32, 32), 0.4 * MM, "hemisphere", 64, 25 * MM, 1024),
    # secondary regime of the paper's Fig. 1f (f_s = 20 MHz, sigma = 62.5 um): W = 5
    "cfg4p": Config("cfg4p", (256, 256, 128), 0.1 * MM, "hemisphere", 1024, 60 * MM, 4096,
                    fs=20e6, sigma=62.5e-6),
}


def random_suite_case(seed):
    """Randomised parity geometry: sigma U[0.05,0.15] mm,
    t0 U[0,5] us, centres jittered +-0.5 dx, hemisphere or planar array,
    ragged grid dims, record length chosen so some windows clip at both ends.
    Returns (centers, sensors, op_kwargs)."""
    rng = np.random.default_rng(1000 + seed)
    dims = tuple(int(v) for v in rng.integers(3, 11, size=3))
    dx = 0.1 * MM
    c = grid_centers(*dims, dx, jitter=0.5, seed=seed)
    sigma = float(rng.uniform(0.05, 0.15)) * MM
    t0 = float(rng.uniform(0.0, 5.0)) * 1e-6
    fs = float(rng.choice([20e6, 40e6, 50e6]))
    v = 1500.0
    if seed % 2 == 0:
        R = float(rng.uniform(8.0, 20.0)) * MM
        s = hemisphere(int(rng.integers(5, 70)), R)
        rmax = R + 1.0 * MM
    else:
        n_side = int(rng.integers(3, 9))
        pitch = float(rng.uniform(1.0, 3.0)) * MM
        s = planar_checkerboard(n_side=n_side, pitch=pitch, z=-float(rng.uniform(3.0, 9.0)) * MM,
                                parity=seed // 2 % 2)
        rmax = float(np.sqrt(((s.astype(np.float64)) ** 2).sum(0)).max()) + 1.0 * MM
    # record ends slightly before the latest window so the tail clips too
    n_samples = int(max(8, ((rmax / v) - t0) * fs * float(rng.uniform(0.9, 1.05))))
    op = dict(sigma=sigma, v=v, fs=fs, n_samples=n_samples, t0=t0, k=3.0)
    return c, s, op


def with_overrides(cfg: Config, **kw):
    return replace(cfg, **kw)
