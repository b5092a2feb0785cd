"""Writes tests/golden/desk_*.{json,npy}: the fp64 oracle's desk-scale
reconstructions -- calls only oracle/ and
the seeded input generators.  Run once (about 5 min on 8 cores):

    python scripts/make_desk_golden.py
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from oracle import ir  # noqa: E402
from paper_2602_03893_b200 import inputs  # noqa: E402

# The two desk cases: noiseless with lambda = 0 and 5:1 amplitude
# noise with the VCR regulariser (row f2 end to end).
CASES = {
    "clean": dict(snr=None, lam=0.0, beta=0.0),
    "noisy": dict(snr=5.0, lam=3e-7, beta=1.0),
}
ITERS = 200
HYPER = dict(eta_min=1e-4, eta_max=0.1, T0=50, Tmult=2, eps_reg=1e-8)


def psnr(a, ref):
    """both max-normalised, psnr = 10 log10(1 / mse)."""
    a = np.asarray(a, np.float64)
    ref = np.asarray(ref, np.float64)
    a = a / np.abs(a).max()
    ref = ref / np.abs(ref).max()
    mse = float(np.mean((a - ref) ** 2))
    return 200.0 if mse < 1e-20 else 10.0 * np.log10(1.0 / mse)


def desk_inputs(case):
    cfg = inputs.CONFIGS["desk"]
    c, s, op = cfg.centers(), cfg.sensors(), cfg.op_kwargs()
    x = inputs.blobs_phantom(*cfg.grid)
    b = oracle.forward(c, x, s, **op).astype(np.float32)
    if CASES[case]["snr"]:
        b = inputs.add_noise(b, CASES[case]["snr"])
    return cfg, c, s, op, x, b


def main():
    out = {}
    for case, p in CASES.items():
        cfg, c, s, op, x, b = desk_inputs(case)
        geom = {"centers": c, "sensors": s, "op": op}
        hp = ir.Hyper(lam=p["lam"], beta=p["beta"], dims=cfg.grid, **HYPER)
        t = time.time()
        xr, st = ir.run(b.astype(np.float64), geom, hp, ITERS)
        bp = oracle.adjoint(c, b, s, **{k: v for k, v in op.items() if k != "n_samples"})
        out[case] = {"iters": ITERS, "lam": p["lam"], "beta": p["beta"], "snr": p["snr"], **HYPER,
                     "losses": st.losses, "psnr": psnr(xr, x), "psnr_single_pass": psnr(bp, x),
                     "seconds": time.time() - t}
        np.save(os.path.join(ROOT, "tests", "golden", f"desk_{case}_x.npy"), xr.astype(np.float32))
        print(case, out[case]["psnr"], out[case]["psnr_single_pass"], out[case]["seconds"], flush=True)
    with open(os.path.join(ROOT, "tests", "golden", "desk_oracle.json"), "w") as f:
        json.dump({"source": "scripts/make_desk_golden.py (oracle/ only)", "cases": out}, f, indent=1)


if __name__ == "__main__":
    main()
