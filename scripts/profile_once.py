"""One forward + one adjoint (+ one iterate) of a config, for ncu captures."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2602_03893_b200 import gpair, inputs

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
assa = len(sys.argv) > 2 and sys.argv[2] == "assa"
cfg = inputs.CONFIGS[name]
dev = torch.device("cuda:0")
ctx = gpair.Context(torch.from_numpy(cfg.centers()).to(dev), torch.from_numpy(cfg.sensors()).to(dev),
                    sigma=cfg.sig, v=cfg.v, fs=cfg.fs, n_samples=cfg.n_samples, t0=cfg.t0, k=cfg.k, assa=assa)
x = torch.from_numpy(inputs.dense_amplitudes(cfg.M)).to(dev)
d = torch.from_numpy(inputs.residual(cfg.n_sensors, cfg.n_samples)).to(dev)
y = ctx.forward(x)
g = ctx.adjoint(d)
z = torch.full_like(x, 0.3); m = torch.zeros_like(x); v = torch.zeros_like(x)
ctx.iterate(z, m, v, y, lr=0.01, step=1)
torch.cuda.synchronize()
print("done", ctx.info())
