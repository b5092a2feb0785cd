"""The ONE parity gate shared by every GPU test (north_star).

For fp32 GPU results against the fp64 oracle -- signals y, gradients g, dL/dz,
Adam state and the one-step update alike:
  * relative L2 error <= 1e-5, and
  * max elementwise relative error <= 1e-4 over the entries with
    |oracle| >= 1e-3 max|oracle|.
There is no looser per-kernel-vector bound.  At the bench sizes the oracle runs
on exact operator rows / columns (32 sampled sensors for forward
rows, 65,536 sampled kernels for adjoint columns).
"""
import numpy as np
import torch

REL_L2 = 1e-5
REL_ELEM = 1e-4
ELEM_FLOOR = 1e-3  # entries gated elementwise: |oracle| >= ELEM_FLOOR * max|oracle|
N_ROWS = 32        # sampled forward rows (sensors) at full size
N_COLS = 65536     # sampled adjoint columns (kernels) at full size


def dev():
    return torch.device("cuda:0")


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev())


def compare(got, ref):
    """(rel L2, max elementwise relative error over |ref| >= ELEM_FLOOR max|ref|)."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    nref = np.linalg.norm(ref)
    rel = np.linalg.norm(got - ref) / nref if nref > 0 else np.linalg.norm(got)
    big = np.abs(ref) >= ELEM_FLOOR * np.abs(ref).max() if nref > 0 else np.zeros(ref.shape, bool)
    elem = float(np.max(np.abs(got[big] - ref[big]) / np.abs(ref[big]))) if big.any() else 0.0
    return rel, elem


def assert_parity(got, ref, what):
    rel, elem = compare(got, ref)
    print(f"{what}: rel L2 {rel:.2e} elementwise {elem:.2e}")
    assert rel <= REL_L2, f"{what}: rel L2 {rel:.3e} > {REL_L2}"
    assert elem <= REL_ELEM, f"{what}: max elementwise rel {elem:.3e} > {REL_ELEM}"
    return rel, elem


def assert_state_update(z_new, z0, z_ref, what):
    """One-step state update z' (Adam or clamp) from z0: the gate on z' itself (SURVEY 8c:
    "the one-step z'"), and rel L2 <= REL_L2 on the step z' - z0 where the fp32 state can
    resolve it.  The step is not gated elementwise: z' carries ulp(z)/2 ~ 3e-8 of rounding,
    ~3e-4 of the smallest gated Adam steps (1e-3 of the largest) whatever the arithmetic."""
    assert_parity(z_new, z_ref, what)
    step, step_ref = np.asarray(z_new, np.float64) - z0, np.asarray(z_ref, np.float64) - z0
    # the fp32 state resolves the step to ~2^-24 |z'| (rms); below REL_L2 of that the step is
    # not representable (e.g. clamp steps with the 2/N gradient scale) and z' is the gate
    quant = 2.0 ** -24 * np.sqrt(np.mean(np.asarray(z_ref, np.float64) ** 2))
    rms = np.sqrt(np.mean(step_ref ** 2))
    if rms < quant / REL_L2:
        print(f"{what}: step rms {rms:.2e} below the fp32 state's resolution; gated through z'")
        return
    rel = np.linalg.norm(step - step_ref) / np.linalg.norm(step_ref)
    print(f"{what} (step z' - z0): rel L2 {rel:.2e}")
    assert rel <= REL_L2, f"{what} step: rel L2 {rel:.3e} > {REL_L2}"


def sample_rows(n_sensors, n=N_ROWS, seed=5):
    """Sorted sensor subset for full-size forward parity (first, last and random rows)."""
    if n_sensors <= n:
        return np.arange(n_sensors, dtype=np.int32)
    rest = np.random.default_rng(seed).choice(np.arange(1, n_sensors - 1), n - 2, replace=False)
    return np.sort(np.concatenate([[0, n_sensors - 1], rest])).astype(np.int32)


def sample_cols(M, n=N_COLS, seed=4):
    """Sorted kernel subset for full-size adjoint parity."""
    if M <= n:
        return np.arange(M, dtype=np.int64)
    return np.sort(np.random.default_rng(seed).choice(M, n, replace=False)).astype(np.int64)


def psnr(a, ref):
    """Desk-scale quality metric: both max-normalised,
    psnr = 10 log10(1 / mse), capped at 200 dB."""
    a = np.asarray(a, np.float64)
    ref = np.asarray(ref, np.float64)
    a = a / np.abs(a).max()
    ref = ref / np.abs(ref).max()
    mse = float(np.mean((a - ref) ** 2))
    return 200.0 if mse < 1e-20 else 10.0 * np.log10(1.0 / mse)
