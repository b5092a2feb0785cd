"""GPU-vs-oracle parity report at SURVEY 8c's sample sizes.

For each config: forward rows (32 sampled sensors, or all when fewer) and
adjoint columns (65,536 sampled kernels, or all when fewer) against the fp64
oracle; prints rel L2, max elementwise relative error over |oracle| >= 1e-3
max|oracle|, how many entries that gate covers, and the error quantiles.
Test infrastructure: calls oracle/ (reporting only; nothing here feeds the
product path).  Usage: python scripts/parity_report.py [cfg ...] [--assa]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
from paper_2602_03893_b200 import gpair, inputs

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from tests_common import N_COLS, N_ROWS, compare, sample_cols, sample_rows  # noqa: E402


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def line(tag, got, ref):
    rel, elem = compare(got, ref)
    ref = np.asarray(ref, np.float64)
    big = np.abs(ref) >= 1e-3 * np.abs(ref).max()
    e = np.abs(np.asarray(got, np.float64)[big] - ref[big]) / np.abs(ref[big])
    q = np.quantile(e, [0.5, 0.99, 0.9999]) if e.size else [0, 0, 0]
    return (f"{tag}: relL2={rel:.3e} elem={elem:.3e} n_gated={int(big.sum())} "
            f"q50={q[0]:.2e} q99={q[1]:.2e} q9999={q[2]:.2e}")


def main(names, assa=False):
    for name in names:
        cfg = inputs.CONFIGS[name]
        c, s, op = cfg.centers(), cfg.sensors(), cfg.op_kwargs()
        kw = dict(sigma=op["sigma"], v=op["v"], fs=op["fs"], n_samples=op["n_samples"], t0=op["t0"], k=op["k"])
        if assa:
            kw["assa"] = True
        ctx = gpair.Context(T(c), T(s), **kw)
        x = inputs.dense_amplitudes(cfg.M)
        d = inputs.residual(cfg.n_sensors, cfg.n_samples)
        y = ctx.forward(T(x)).cpu().numpy()
        g = ctx.adjoint(T(d)).cpu().numpy()
        rows, cols = sample_rows(cfg.n_sensors), sample_cols(cfg.M)
        akw = {k: v for k, v in op.items() if k != "n_samples"}
        t = time.perf_counter()
        cache = f"/tmp/parity_oracle_{name}_{int(assa)}_{len(rows)}_{len(cols)}.npz"
        if os.path.exists(cache):  # the oracle's rows / columns, reused across library variants
            z = np.load(cache)
            yr, gr = z["yr"], z["gr"]
        elif assa:
            p = oracle.assa_params(op["sigma"], op["v"], op["fs"], op["k"], 25)
            yr = oracle.assa_forward(c, x, s, rows=rows, alpha=p["alpha"], K=p["K"], **op)
            gr = oracle.assa_adjoint(c, d, s, cols=cols, alpha=p["alpha"], K=p["K"], **akw)
        else:
            yr = oracle.forward(c, x, s, rows=rows, **op)
            gr = oracle.adjoint(c, d, s, cols=cols, **akw)
        if not os.path.exists(cache):
            np.savez(cache, yr=yr, gr=gr)
        to = time.perf_counter() - t
        lib = os.environ.get("GPAIR_LIB", "libgpair.so")
        print(f"[{lib}] {name}{' assa' if assa else ''} rows={len(rows)} cols={len(cols)} (oracle {to:.1f} s)")
        print("  " + line("forward rows", y[rows], yr))
        print("  " + line("adjoint cols", g[cols], gr), flush=True)
        ctx.close()


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    main(args or ["cfg1", "cfg2", "cfg4"], assa="--assa" in sys.argv)
