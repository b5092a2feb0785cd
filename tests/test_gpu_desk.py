"""Desk-scale reconstruction workload on the GPU (PAPER.md
Alg. 2; SPEC acceptance S:732-735 used as test ideas).

32^3 kernels at 0.4 mm, 64-element hemisphere, 5-blob phantom, oracle data,
200 iterations of `gpair_iterate` through `recon.reconstruct`:
  * quality: PSNR >= 28 dB and >= 6 dB over the single-pass A^T b (S:732a-b);
  * x >= 0 exactly (NPC) and loss drop >= 100x (S:732c-d);
  * 5:1 amplitude noise with the VCR regulariser (row f2): PSNR >= 22 dB;
  * determinism: two runs are bit-identical;
  * against the fp64 oracle's own 200-iteration runs (tests/golden/
    desk_oracle.json + desk_*_x.npy, written by scripts/make_desk_golden.py
    from oracle/ only): the first loss to 1e-5 (same z = 0 start), the loss
    trajectory and final PSNR within reported fp32-drift bounds (reading R12).
"""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from paper_2602_03893_b200 import gpair, inputs, recon  # noqa: E402

from tests_common import T, dev, psnr  # noqa: E402

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_03893_b200 import build

    build.build()


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(GOLDEN, "desk_oracle.json")) as f:
        return json.load(f)["cases"]


@pytest.fixture(scope="module")
def desk():
    cfg = inputs.CONFIGS["desk"]
    c, s, op = cfg.centers(), cfg.sensors(), cfg.op_kwargs()
    x_true = inputs.blobs_phantom(*cfg.grid)
    b = oracle.forward(c, x_true, s, **op).astype(np.float32)
    ctx = gpair.Context(T(c), T(s), sigma=op["sigma"], v=op["v"], fs=op["fs"], n_samples=op["n_samples"],
                        t0=op["t0"], k=op["k"])
    return cfg, ctx, x_true, b


def _sched(g):
    return recon.Schedule(iters=g["iters"], eta_min=g["eta_min"], eta_max=g["eta_max"], T0=g["T0"],
                          Tmult=g["Tmult"], lam=g["lam"], beta=g["beta"], eps_reg=g["eps_reg"])


def _run(ctx, b, g, grid):
    x, losses = recon.reconstruct(ctx, T(b), _sched(g), grid=grid)
    torch.cuda.synchronize()
    return x, losses


def test_desk_clean_quality_and_oracle_agreement(desk, golden):
    cfg, ctx, x_true, b = desk
    g = golden["clean"]
    x, losses = _run(ctx, b, g, cfg.grid)
    xh, lh = x.cpu().numpy(), losses.cpu().numpy()
    p = psnr(xh, x_true)
    bp = ctx.adjoint(T(b)).cpu().numpy()
    p1 = psnr(bp, x_true)
    lo = np.array(g["losses"])
    x_or = np.load(os.path.join(GOLDEN, "desk_clean_x.npy"))
    print(f"desk clean: PSNR {p:.2f} dB (oracle {g['psnr']:.2f}), single pass {p1:.2f} dB "
          f"(oracle {g['psnr_single_pass']:.2f}), loss {lh[0]:.4e} -> {lh[-1]:.4e}, "
          f"PSNR(gpu vs oracle x) {psnr(xh, x_or):.1f} dB, max traj rel {np.max(np.abs(lh - lo) / lo):.2e}")
    assert p >= 28.0
    assert p - p1 >= 6.0
    assert np.all(xh >= 0.0)
    assert lh[-1] < 1e-2 * lh[0]
    assert abs(lh[0] - lo[0]) <= 1e-5 * lo[0]
    assert np.max(np.abs(lh[:20] - lo[:20]) / lo[:20]) < 1e-2
    assert abs(p - g["psnr"]) <= 1.0
    assert abs(p1 - g["psnr_single_pass"]) <= 1e-3


def test_desk_noisy_with_vcr(desk, golden):
    cfg, ctx, x_true, b = desk
    g = golden["noisy"]
    bn = inputs.add_noise(b, g["snr"])
    x, losses = _run(ctx, bn, g, cfg.grid)
    xh, lh = x.cpu().numpy(), losses.cpu().numpy()
    p = psnr(xh, x_true)
    lo = np.array(g["losses"])
    print(f"desk noisy+VCR: PSNR {p:.2f} dB (oracle {g['psnr']:.2f}), loss {lh[0]:.4e} -> {lh[-1]:.4e}")
    assert p >= 22.0
    assert np.all(xh >= 0.0)
    assert abs(lh[0] - lo[0]) <= 1e-5 * lo[0]
    assert abs(p - g["psnr"]) <= 1.0


def test_desk_deterministic(desk, golden):
    cfg, ctx, _, b = desk
    g = dict(golden["noisy"], iters=60)
    x1, l1 = _run(ctx, b, g, cfg.grid)
    x2, l2 = _run(ctx, b, g, cfg.grid)
    assert torch.equal(x1, x2) and torch.equal(l1, l2)
