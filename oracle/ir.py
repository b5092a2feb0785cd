"""Algorithm 2 (GPAIR loop) in plain numpy fp64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Each function follows the
paper in its own order and notation:

* NPC (Eq. 18):   x = phi(z) = (z + eps)^2,  eps = 1e-8
* chain rule (Eq. 19):  dL/dz = dL/dx * 2 (z + eps)
* loss (Eq. 23):  L = (1/N) ||A(phi(z)) - b||^2 + lambda R_VCR(x),
  N = N_d N_t; R_VCR (Eqs. 20-22, row f2) in oracle/vcr.py, lambda = 0 default.
* gradient scale (reading R10): dL/dy = (2/N)(y - b); ``grad_scale`` exposed,
  1.0 reproduces Alg. 2 line 529 literally.
* CAWR (Eq. 24), as printed by default (reading R13).
* Adam (reading R11): beta1=0.9, beta2=0.999, eps_a=1e-8,
  bias-corrected, no weight decay:
      m = b1 m + (1-b1) g;  v = b2 v + (1-b2) g^2
      m_hat = m / (1 - b1^t);  v_hat = v / (1 - b2^t)   (t = iteration + 1)
      z = z - eta_t * m_hat / (sqrt(v_hat) + eps_a)
* clamp mode (reading R15, north_star "non-negativity clamp"):
      x = max(x - eta_t * dL/dx, 0), state is x itself.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import adjoint as _adjoint
from . import assa_adjoint as _assa_adjoint
from . import assa_forward as _assa_forward
from . import forward as _forward

EPS_NPC = 1e-8


def npc(z, eps=EPS_NPC):
    """Eq. 18: x = (z + eps)^2."""
    return (z + eps) ** 2


def npc_chain(grad_x, z, eps=EPS_NPC):
    """Eq. 19: dL/dz = dL/dx (.) 2 (z + eps)."""
    return grad_x * (2.0 * (z + eps))


def cawr(t, eta_min, eta_max, T0, Tmult=1, printed_formula=True):
    """Eq. 24.

    printed_formula=True: T_cur = t mod T0, T_i = T0 * Tmult^floor(t/T0) exactly
    as printed.  False: the SGDR schedule of the cited ref. (restart after each
    geometric period), which coincides with the printed one for Tmult = 1.
    """
    if printed_formula or Tmult == 1:
        T_cur = t % T0
        T_i = T0 * Tmult ** (t // T0)
    else:
        n = int(math.floor(math.log(t / T0 * (Tmult - 1) + 1, Tmult)))
        start = T0 * (Tmult ** n - 1) // (Tmult - 1)
        T_cur = t - start
        T_i = T0 * Tmult ** n
    return eta_min + 0.5 * (eta_max - eta_min) * (1.0 + math.cos(math.pi * T_cur / T_i))


@dataclass
class Hyper:
    eta_min: float = 1e-4
    eta_max: float = 0.1
    T0: int = 50
    Tmult: int = 1
    beta1: float = 0.9
    beta2: float = 0.999
    adam_eps: float = 1e-8
    eps_npc: float = EPS_NPC
    grad_scale: float | None = None  # None -> 2/N
    mode: str = "npc"  # "npc" (paper) | "clamp"
    printed_formula: bool = True
    lam: float = 0.0  # lambda of Eq. 23 (VCR weight, row f2)
    beta: float = 0.0  # beta of Eq. 20
    eps_reg: float = 1e-8  # regulariser epsilon (reading V4)
    dims: tuple | None = None  # voxel grid (nx, ny, nz) of the kernel order, needed when lam > 0


@dataclass
class State:
    z: np.ndarray
    m: np.ndarray
    v: np.ndarray
    t: int = 0  # iterations done
    losses: list = field(default_factory=list)


def init_state(M):
    """Alg. 2: z^(0) = 0, m = v = 0."""
    return State(z=np.zeros(M), m=np.zeros(M), v=np.zeros(M))


def data_loss(y, b):
    """Eq. 23 data term (1/N)||y - b||^2, N = N_d * N_t."""
    r = y - b
    return float(np.sum(r * r) / r.size)


def loss_and_grad(z, b, geom, hp: Hyper):
    """L(z) and dL/dz for lambda = 0 (Alg. 2)."""
    x = npc(z, hp.eps_npc) if hp.mode == "npc" else z
    assa = geom.get("assa")  # {"alpha", "K"}: the ASSA operator (row f1) instead of Eq. 7
    if assa:
        y = _assa_forward(geom["centers"], x, geom["sensors"], **geom["op"], **assa)
    else:
        y = _forward(geom["centers"], x, geom["sensors"], **geom["op"])
    r = y - b
    N = r.size
    L = float(np.sum(r * r) / N)
    scale = (2.0 / N) if hp.grad_scale is None else hp.grad_scale
    if assa:
        gx = _assa_adjoint(geom["centers"], scale * r, geom["sensors"], **_adj_kw(geom["op"]), **assa)
    else:
        gx = _adjoint(geom["centers"], scale * r, geom["sensors"], **_adj_kw(geom["op"]))
    if hp.lam > 0.0:  # Alg. 2: L += lambda R_VCR(x), grad_x += lambda grad R_VCR(x)
        from .vcr import r_vcr

        rv, gv = r_vcr(x, hp.dims, hp.beta, hp.eps_reg)
        L += hp.lam * rv
        gx = gx + hp.lam * gv
    gz = npc_chain(gx, z, hp.eps_npc) if hp.mode == "npc" else gx
    return L, gz, y


def _adj_kw(op):
    return {k: v for k, v in op.items() if k != "n_samples"}


def adam_update(z, m, v, g, lr, t1, hp: Hyper):
    """One bias-corrected Adam step; t1 = 1-based step count."""
    m = hp.beta1 * m + (1.0 - hp.beta1) * g
    v = hp.beta2 * v + (1.0 - hp.beta2) * g * g
    m_hat = m / (1.0 - hp.beta1 ** t1)
    v_hat = v / (1.0 - hp.beta2 ** t1)
    z = z - lr * m_hat / (np.sqrt(v_hat) + hp.adam_eps)
    return z, m, v


def step(state: State, b, geom, hp: Hyper):
    """One iteration t of Algorithm 2. Returns (loss, y)."""
    t = state.t
    L, gz, y = loss_and_grad(state.z, b, geom, hp)
    lr = cawr(t, hp.eta_min, hp.eta_max, hp.T0, hp.Tmult, hp.printed_formula)
    if hp.mode == "npc":
        state.z, state.m, state.v = adam_update(state.z, state.m, state.v, gz, lr, t + 1, hp)
    else:
        state.z = np.maximum(state.z - lr * gz, 0.0)
    state.t = t + 1
    state.losses.append(L)
    return L, y


def run(b, geom, hp: Hyper, iters, state=None):
    """Algorithm 2 end to end; returns (x*, state). x* = (z + eps)^2 (line 539)."""
    M = geom["centers"].shape[1]
    state = state or init_state(M)
    for _ in range(iters):
        step(state, b, geom, hp)
    x = npc(state.z, hp.eps_npc) if hp.mode == "npc" else state.z
    return x, state
