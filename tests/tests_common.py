"""Helpers shared by the GPU parity tests (tolerances: north_star / DESIGN.md R19)."""
import numpy as np
import torch

REL_L2 = 1e-5
REL_ELEM = 1e-4


def dev():
    return torch.device("cuda:0")


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev())


def compare(got, ref):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    nref = np.linalg.norm(ref)
    rel = np.linalg.norm(got - ref) / nref if nref > 0 else np.linalg.norm(got)
    big = np.abs(ref) >= 1e-3 * np.abs(ref).max() if nref > 0 else np.zeros(ref.shape, bool)
    elem = float(np.max(np.abs(got[big] - ref[big]) / np.abs(ref[big]))) if big.any() else 0.0
    return rel, elem


def assert_parity(got, ref, what, elementwise=True):
    """rel L2 gate on everything; the elementwise gate applies to signal
    samples (north_star: "1e-4 max elementwise relative error on samples
    above 1e-3 of peak"; reading R19).  For per-kernel vectors it
    is reported with a 10x looser sanity bound."""
    rel, elem = compare(got, ref)
    assert rel <= REL_L2, f"{what}: rel L2 {rel:.3e}"
    bound = REL_ELEM if elementwise else 10 * REL_ELEM
    assert elem <= bound, f"{what}: max elementwise rel {elem:.3e}"
    return rel, elem




def psnr(a, ref):
    """Desk-scale quality metric: both max-normalised,
    psnr = 10 log10(1 / mse), capped at 200 dB."""
    a = np.asarray(a, np.float64)
    ref = np.asarray(ref, np.float64)
    a = a / np.abs(a).max()
    ref = ref / np.abs(ref).max()
    mse = float(np.mean((a - ref) ** 2))
    return 200.0 if mse < 1e-20 else 10.0 * np.log10(1.0 / mse)
