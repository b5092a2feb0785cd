"""Print gpair_get_info for a config (which kernel paths it takes)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_03893_b200 import gpair, inputs

for name in sys.argv[1:]:
    cfg = inputs.CONFIGS[name]
    ctx = gpair.Context(torch.from_numpy(cfg.centers()).cuda(), torch.from_numpy(cfg.sensors()).cuda(), sigma=cfg.sig,
                        v=cfg.v, fs=cfg.fs, n_samples=cfg.n_samples, t0=cfg.t0, k=cfg.k)
    print(name, ctx.info(), flush=True)
    ctx.close()
