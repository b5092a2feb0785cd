"""Print GPU-vs-oracle errors (rel L2, max elementwise over |ref| >= 1e-3 peak)
for cfg1 (full) and sampled rows / columns of cfg2 and cfg4, plus forward /
adjoint kernel times.  Test infrastructure: calls oracle/ (allowed in scripts
that only report; nothing here feeds the product path)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
from paper_2602_03893_b200 import gpair, inputs


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def compare(got, ref):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    big = np.abs(ref) >= 1e-3 * np.abs(ref).max()
    return rel, float(np.max(np.abs(got[big] - ref[big]) / np.abs(ref[big])))


def timed(fn, n=3):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / n * 1e3


def main(names):
    for name in names:
        cfg = inputs.CONFIGS[name]
        c, s, op = cfg.centers(), cfg.sensors(), cfg.op_kwargs()
        ctx = gpair.Context(T(c), T(s), sigma=op["sigma"], v=op["v"], fs=op["fs"], n_samples=op["n_samples"],
                            t0=op["t0"], k=op["k"])
        x = inputs.dense_amplitudes(cfg.M)
        xt = T(x)
        d = inputs.residual(cfg.n_sensors, cfg.n_samples)
        dt = T(d)
        y = ctx.forward(xt).cpu().numpy()
        g = ctx.adjoint(dt).cpu().numpy()
        akw = {k: v for k, v in op.items() if k != "n_samples"}
        if cfg.M * cfg.n_sensors <= 5e6:
            ey = compare(y, oracle.forward(c, x, s, **op))
            eg = compare(g, oracle.adjoint(c, d, s, **akw))
        else:
            rows = np.array(sorted({0, 1, cfg.n_sensors // 3, cfg.n_sensors // 2, cfg.n_sensors - 1}), np.int32)
            ey = compare(y[rows], oracle.forward(c, x, s, rows=rows, **op))
            cols = np.random.default_rng(4).choice(cfg.M, 2048, replace=False).astype(np.int64)
            eg = compare(g[cols], oracle.adjoint(c, d, s, cols=cols, **akw))
        tf = timed(lambda: ctx.forward(xt))
        ta = timed(lambda: ctx.adjoint(dt))
        print(f"{name} tab={os.environ.get('GPAIR_NO_TAB', '0') != '1'}: forward relL2={ey[0]:.3e} elem={ey[1]:.3e} "
              f"| adjoint relL2={eg[0]:.3e} elem={eg[1]:.3e} | fwd {tf:.2f} ms adj {ta:.2f} ms", flush=True)
        ctx.close()


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg1", "cfg2", "cfg4"])
