"""Algorithm 2 end to end on the GPU: the
reconstruction loop a user calls, built only from the library's C-ABI
(`gpair_iterate` per iteration, `gpair_cawr_lr` for Eq. 24's schedule).

SURVEY 8f row f3 drives it on the desk-scale workload; bench.py times one
`gpair_iterate` of the same loop.  There is no CPU path: without the CUDA
library `gpair.lib()` raises.
"""
from __future__ import annotations

from dataclasses import dataclass

from . import gpair


@dataclass
class Schedule:
    """Alg. 2 hyper-parameters (readings R11, R13, R14; V4)."""
    iters: int = 200
    eta_min: float = 1e-4
    eta_max: float = 0.1
    T0: int = 50
    Tmult: int = 1
    printed_formula: bool = True
    mode: int = 0  # 0 = NPC + Adam (paper), 1 = projected clamp (R15)
    lam: float = 0.0  # lambda of Eq. 23
    beta: float = 0.0  # beta of Eq. 20
    eps_reg: float = 1e-8
    eps_npc: float = 1e-8
    grad_scale: float = 0.0  # dL/dy = grad_scale (y - b); <= 0 -> 2/N (R10); 1.0 = Alg. 2 line 529 literally


def reconstruct(ctx: gpair.Context, b, sched: Schedule, grid=None, stream=None):
    """Runs `sched.iters` iterations from z = 0, m = v = 0 (Alg. 2 lines
    514-515).  b: CUDA float32 [N_d][N_t].  Returns (x, losses): x = the
    final image (z + eps)^2 (line 539) as a CUDA tensor [M], losses a CUDA
    tensor [iters] of L(z_t) recorded without host synchronisation."""
    import torch

    if sched.iters < 1:
        raise ValueError("iters must be >= 1")
    if sched.lam > 0 and grid is None:
        raise ValueError("lam > 0 needs the voxel grid (nx, ny, nz)")
    dev = b.device
    z = torch.zeros(ctx.M, device=dev)
    m = torch.zeros_like(z)
    v = torch.zeros_like(z)
    x = torch.empty_like(z)
    losses = torch.empty(sched.iters, device=dev)
    for t in range(sched.iters):
        lr = gpair.cawr_lr(t, sched.eta_min, sched.eta_max, sched.T0, sched.Tmult, sched.printed_formula)
        ctx.iterate(z, m, v, b, lr=lr, step=t + 1, mode=sched.mode, eps_npc=sched.eps_npc, grad_scale=sched.grad_scale,
                    lam=sched.lam,
                    beta=sched.beta, eps_reg=sched.eps_reg, grid=grid,
                    x_out=x if t == sched.iters - 1 else None, loss_out=losses[t:t + 1], stream=stream)
    return x, losses
