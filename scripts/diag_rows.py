"""Diagnostics: GPU vs oracle forward rows for a config; saves both to gpurun_out/diag_<cfg>.npz."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle
from paper_2602_03893_b200 import gpair, inputs

name = sys.argv[1]
cfg = inputs.CONFIGS[name]
c, s, op = cfg.centers(), cfg.sensors(), cfg.op_kwargs()
ctx = gpair.Context(torch.from_numpy(c).cuda(), torch.from_numpy(s).cuda(), sigma=op["sigma"], v=op["v"], fs=op["fs"],
                    n_samples=op["n_samples"], t0=op["t0"], k=op["k"])
x = inputs.dense_amplitudes(cfg.M)
y = ctx.forward(torch.from_numpy(x).cuda()).cpu().numpy()
rows = np.array(sorted({0, 1, cfg.n_sensors // 3, cfg.n_sensors // 2, cfg.n_sensors - 1}), np.int32)
ref = oracle.forward(c, x, s, rows=rows, **op)
# |terms| sum: forward of |a_ijn| is not available; use x = 1 on a sign-split: sum of positive and negative parts
np.savez_compressed(f"gpurun_out/diag_{name}.npz", got=y[rows], ref=ref, rows=rows)
print("saved", rows)
