"""Thin ctypes binding of libgpair.so (include/gpair.h) -- argument marshalling only.

Every step of the hot path runs in the CUDA kernels behind the C ABI; this
module only converts torch CUDA tensors to device pointers and the current
torch stream to a cudaStream_t.  There is no CPU fallback: if the library is
missing or no CUDA device is present, calls raise.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, os.environ.get("GPAIR_LIB", "libgpair.so"))

OK, ERR_INVALID_ARGUMENT, ERR_GEOMETRY, ERR_RESOURCE, ERR_NUMERICAL, ERR_CUDA, ERR_NCCL = range(7)
CHECK_FINITE = 1 << 9
TOF_ASSA = 1
NEAR_FIELD = 1 << 1
COLLECTIVE = 1 << 2
PROF_NAMES = ["gather", "forward", "reduce", "allreduce", "residual", "adjoint", "loss", "vcr"]


class GpairError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"gpair status {status}: {msg}")
        self.status = status


class Desc(ctypes.Structure):
    _fields_ = [
        ("sound_speed", ctypes.c_double),
        ("sampling_rate", ctypes.c_double),
        ("n_samples", ctypes.c_int32),
        ("t0", ctypes.c_double),
        ("n_kernels", ctypes.c_int64),
        ("centers", ctypes.c_void_p),
        ("sigma", ctypes.c_double),
        ("sigmas", ctypes.c_void_p),
        ("window_k", ctypes.c_double),
        ("n_sensors", ctypes.c_int32),
        ("sensors", ctypes.c_void_p),
        ("rank", ctypes.c_int32),
        ("world", ctypes.c_int32),
        ("nccl_comm", ctypes.c_void_p),
        ("flags", ctypes.c_int32),
        ("assa_nmin", ctypes.c_int32),
    ]


class Step(ctypes.Structure):
    _fields_ = [
        ("lr", ctypes.c_float),
        ("beta1", ctypes.c_float),
        ("beta2", ctypes.c_float),
        ("adam_eps", ctypes.c_float),
        ("eps_npc", ctypes.c_float),
        ("grad_scale", ctypes.c_float),
        ("step", ctypes.c_int32),
        ("mode", ctypes.c_int32),
        ("lam", ctypes.c_float),
        ("beta", ctypes.c_float),
        ("eps_reg", ctypes.c_float),
        ("grid", ctypes.c_int32 * 3),
        ("z0", ctypes.c_int32),
    ]


class Profile(ctypes.Structure):
    _fields_ = [("ms", ctypes.c_double * len(PROF_NAMES)), ("launches", ctypes.c_int64 * len(PROF_NAMES)),
                ("kernels", ctypes.c_int64)]


class Info(ctypes.Structure):
    _fields_ = [
        ("n_kernels", ctypes.c_int64),
        ("n_kernels_padded", ctypes.c_int64),
        ("n_cells", ctypes.c_int32),
        ("fwd_region_cells", ctypes.c_int32),
        ("fwd_regions", ctypes.c_int32),
        ("fwd_window", ctypes.c_int32),
        ("fwd_warps", ctypes.c_int32),
        ("adj_region_cells", ctypes.c_int32),
        ("adj_regions", ctypes.c_int32),
        ("adj_window", ctypes.c_int32),
        ("wmax", ctypes.c_int32),
        ("grid_detected", ctypes.c_int32),
        ("max_eps", ctypes.c_double),
        ("workspace_bytes", ctypes.c_int64),
        ("assa", ctypes.c_int32),
        ("assa_alpha", ctypes.c_int32),
        ("assa_n_half", ctypes.c_int32),
        ("assa_K", ctypes.c_int32),
        ("general", ctypes.c_int32),
        ("near_rows", ctypes.c_int32),
        ("near_pairs", ctypes.c_int64),
        ("tab", ctypes.c_int32),
        ("adj_kernel", ctypes.c_int32),
        ("collective", ctypes.c_int32),
        ("fwd_union", ctypes.c_int32),
        ("adj_fit_err", ctypes.c_double),
        ("adj_row_bytes", ctypes.c_int32),
    ]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_lib = None


def lib():
    """Load libgpair.so (built by __graft_entry__.build()); raise if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build() (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64, d = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        st = ctypes.c_int
        sigs = {
            "gpair_create": (st, [ctypes.POINTER(vp), ctypes.POINTER(Desc), vp]),
            "gpair_forward": (st, [vp, vp, vp, vp]),
            "gpair_adjoint": (st, [vp, vp, vp, vp]),
            "gpair_iterate": (st, [vp, vp, vp, vp, vp, ctypes.POINTER(Step), vp, vp, vp, vp]),
            "gpair_count_pair_samples": (st, [vp, ctypes.POINTER(i64), vp]),
            "gpair_vcr": (st, [vp, ctypes.POINTER(i32), vp, ctypes.c_float, ctypes.c_float, vp, vp, vp]),
            "gpair_vcr_slab": (st, [vp, ctypes.POINTER(i32), i32, i32, vp, i32, i32, ctypes.c_float, ctypes.c_float,
                                    vp, vp, vp]),
            "gpair_vcr_prepare": (st, [vp, ctypes.POINTER(i32), i32, vp]),
            "gpair_get_info": (st, [vp, ctypes.POINTER(Info)]),
            "gpair_destroy": (st, [vp]),
            "gpair_profile_enable": (st, [vp, ctypes.c_int]),
            "gpair_profile_read": (st, [vp, ctypes.POINTER(Profile)]),
            "gpair_cawr_lr": (d, [i64, d, d, i64, i64, ctypes.c_int]),
            "gpair_nccl_unique_id": (st, [vp]),
            "gpair_nccl_comm_init": (st, [ctypes.POINTER(vp), i32, vp, i32]),
            "gpair_nccl_comm_destroy": (st, [vp]),
            "gpair_strerror": (ctypes.c_char_p, [st]),
            "gpair_last_error": (ctypes.c_char_p, [vp]),
            "gpair_version": (ctypes.c_char_p, []),
        }
        for name, (res, args) in sigs.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(status, ctx=None):
    if status != OK:
        L = lib()
        raise GpairError(status, f"{L.gpair_strerror(status).decode()}: {L.gpair_last_error(ctx).decode()}")


def _ptr(t, dtype=None, numel=None, name="tensor"):
    """Device pointer of a contiguous float32 CUDA tensor (validated)."""
    import torch

    if t is None:
        return None
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA torch.Tensor")
    if t.dtype != (dtype or torch.float32):
        raise TypeError(f"{name} must be {dtype or torch.float32}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if numel is not None and t.numel() != numel:
        raise ValueError(f"{name} must have {numel} elements, got {t.numel()}")
    return t.data_ptr()


def _stream(stream):
    import torch

    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def cawr_lr(t, eta_min, eta_max, T0, Tmult=1, printed_formula=True):
    """Eq. 24 (host function of the library)."""
    return lib().gpair_cawr_lr(int(t), float(eta_min), float(eta_max), int(T0), int(Tmult), int(bool(printed_formula)))


def version():
    return lib().gpair_version().decode()


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().gpair_nccl_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
    return buf.raw


def nccl_comm_init(world, uid: bytes, rank):
    comm = ctypes.c_void_p()
    buf = ctypes.create_string_buffer(uid, 128)
    _check(lib().gpair_nccl_comm_init(ctypes.byref(comm), int(world), ctypes.cast(buf, ctypes.c_void_p), int(rank)))
    return comm.value


def nccl_comm_destroy(comm):
    _check(lib().gpair_nccl_comm_destroy(comm))


class Context:
    """One gpair_ctx (one rank / device).  Mirrors include/gpair.h."""

    def __init__(self, centers, sensors, *, sigma, v, fs, n_samples, t0=0.0, k=3.0, rank=0, world=1,
                 nccl_comm=None, flags=0, assa=False, assa_nmin=25, sigmas=None, near_field=False, stream=None):
        """sigmas: optional CUDA float32 [M] per-kernel sigma_i (row f4);
        near_field: Eq. 6 with both terms (GPAIR_NEAR_FIELD, row f4)."""
        self.M = int(centers.shape[1])
        self.Nd = int(sensors.shape[1])
        self.Nt = int(n_samples)
        flags = int(flags) | (TOF_ASSA if assa else 0) | (NEAR_FIELD if near_field else 0)
        d = Desc(sound_speed=float(v), sampling_rate=float(fs), n_samples=self.Nt, t0=float(t0),
                 n_kernels=self.M, centers=_ptr(centers, numel=3 * self.M, name="centers"), sigma=float(sigma),
                 sigmas=_ptr(sigmas, numel=self.M, name="sigmas"), window_k=float(k), n_sensors=self.Nd,
                 sensors=_ptr(sensors, numel=3 * self.Nd, name="sensors"), rank=int(rank), world=int(world),
                 nccl_comm=nccl_comm, flags=flags, assa_nmin=int(assa_nmin))
        h = ctypes.c_void_p()
        st = lib().gpair_create(ctypes.byref(h), ctypes.byref(d), _stream(stream))
        _check(st, None)
        self._h = h

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            lib().gpair_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def forward(self, amplitudes, out=None, stream=None):
        import torch

        if out is None:
            out = torch.empty((self.Nd, self.Nt), dtype=torch.float32, device=amplitudes.device)
        _check(lib().gpair_forward(self._h, _ptr(amplitudes, numel=self.M, name="amplitudes"),
                                   _ptr(out, numel=self.Nd * self.Nt, name="signals"), _stream(stream)), self._h)
        return out

    def adjoint(self, residual, out=None, stream=None):
        import torch

        if out is None:
            out = torch.empty(self.M, dtype=torch.float32, device=residual.device)
        _check(lib().gpair_adjoint(self._h, _ptr(residual, numel=self.Nd * self.Nt, name="residual"),
                                   _ptr(out, numel=self.M, name="grad"), _stream(stream)), self._h)
        return out

    def iterate(self, z, m, v, b, *, lr, step, mode=0, beta1=0.9, beta2=0.999, adam_eps=1e-8, eps_npc=1e-8,
                grad_scale=0.0, lam=0.0, beta=0.0, eps_reg=1e-8, grid=None, z0=0, signals_out=None, x_out=None,
                loss_out=None, stream=None):
        """One Alg. 2 iteration; lam > 0 adds lam R_VCR (Eqs. 20-23) over the
        voxel grid `grid` = (nx, ny, nz) of the kernel order; at world > 1
        `grid` is the global grid and `z0` this rank's first z plane."""
        g3 = (ctypes.c_int32 * 3)(*(grid if grid is not None else (0, 0, 0)))
        s = Step(lr=lr, beta1=beta1, beta2=beta2, adam_eps=adam_eps, eps_npc=eps_npc, grad_scale=grad_scale,
                 step=int(step), mode=int(mode), lam=lam, beta=beta, eps_reg=eps_reg, grid=g3, z0=int(z0))
        n = self.M
        _check(lib().gpair_iterate(self._h, _ptr(z, numel=n, name="z"), _ptr(m, numel=n, name="m"),
                                   _ptr(v, numel=n, name="v"), _ptr(b, numel=self.Nd * self.Nt, name="b"),
                                   ctypes.byref(s), _ptr(signals_out, numel=self.Nd * self.Nt, name="signals_out"),
                                   _ptr(x_out, numel=n, name="x_out"), _ptr(loss_out, numel=1, name="loss_out"),
                                   _stream(stream)), self._h)

    def vcr(self, x, grid, *, beta, eps=1e-8, grad=None, value=None, stream=None):
        """R_VCR(x) = R_H + beta R_TV (Eqs. 20-22) into device `value` [1]
        and/or its gradient into device `grad` [prod(grid)]."""
        n = int(grid[0]) * int(grid[1]) * int(grid[2])
        g3 = (ctypes.c_int32 * 3)(*(int(d) for d in grid))
        n = n if n > 0 else None  # bad grids are rejected by the library (INVALID_ARGUMENT)
        _check(lib().gpair_vcr(self._h, g3, _ptr(x, numel=n, name="x"), float(beta), float(eps),
                               _ptr(grad, numel=n, name="grad"), _ptr(value, numel=1, name="value"),
                               _stream(stream)), self._h)

    def vcr_slab(self, x_ext, grid, z0, nz_own, ext_z0, *, beta, eps=1e-8, grad=None, value=None, stream=None):
        """R_VCR's own-plane part of the z slab [z0, z0 + nz_own) of the global
        grid (gpair_vcr_slab): x_ext holds the planes from ext_z0 (the slab and
        its halos), grad gets [nx ny nz_own] entries, value the slab's share."""
        P = int(grid[0]) * int(grid[1])
        ext_nz = int(x_ext.numel()) // P if P > 0 else 0
        g3 = (ctypes.c_int32 * 3)(*(int(d) for d in grid))
        _check(lib().gpair_vcr_slab(self._h, g3, int(z0), int(nz_own), _ptr(x_ext, name="x_ext"), int(ext_z0), ext_nz,
                                    float(beta), float(eps), _ptr(grad, numel=P * int(nz_own), name="grad"),
                                    _ptr(value, numel=1, name="value"), _stream(stream)), self._h)

    def vcr_prepare(self, grid, z0=0, stream=None):
        """gpair_vcr_prepare: agree on / allocate the R_VCR slab layout (collective
        on the collective path: every rank calls it)."""
        g3 = (ctypes.c_int32 * 3)(*(int(d) for d in grid))
        _check(lib().gpair_vcr_prepare(self._h, g3, int(z0), _stream(stream)), self._h)

    def count_pair_samples(self, stream=None):
        out = ctypes.c_int64()
        _check(lib().gpair_count_pair_samples(self._h, ctypes.byref(out), _stream(stream)), self._h)
        return out.value

    def info(self):
        i = Info()
        _check(lib().gpair_get_info(self._h, ctypes.byref(i)), self._h)
        return i.as_dict()

    def profile_enable(self, on=True):
        _check(lib().gpair_profile_enable(self._h, int(bool(on))), self._h)

    def profile_read(self):
        p = Profile()
        _check(lib().gpair_profile_read(self._h, ctypes.byref(p)), self._h)
        return {name: (p.ms[i], p.launches[i]) for i, name in enumerate(PROF_NAMES)}

    def profile_kernels(self):
        """Library kernels launched by the per-call entry points since profile_enable()."""
        p = Profile()
        _check(lib().gpair_profile_read(self._h, ctypes.byref(p)), self._h)
        return int(p.kernels)
