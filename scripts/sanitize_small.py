"""Small runs of every kernel path for compute-sanitizer (memcheck / racecheck / synccheck):
TAB forward + moment-polynomial (TMA / mbarrier ring) / LCF / sensor-lane / lane-per-kernel adjoints, the per-sample path, iterate
(NPC + clamp), ASSA, VCR and the near-field operator, on tiny instances."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2602_03893_b200 import gpair, inputs


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def run(c, s, op, **kw):
    ctx = gpair.Context(T(c), T(s), sigma=op["sigma"], v=op["v"], fs=op["fs"], n_samples=op["n_samples"],
                        t0=op["t0"], k=op["k"], **kw)
    M, Nd = c.shape[1], s.shape[1]
    x = T(inputs.dense_amplitudes(M))
    y = ctx.forward(x)
    g = ctx.adjoint(T(inputs.residual(Nd, op["n_samples"])))
    for mode in (0, 1):
        z = torch.full((M,), 0.3, device="cuda")
        m = torch.zeros_like(z)
        v = torch.zeros_like(z)
        ctx.iterate(z, m, v, y, lr=0.01, step=1, mode=mode)
    torch.cuda.synchronize()
    info = ctx.info()
    ctx.close()
    return info


c = inputs.grid_centers(8, 8, 8, 1e-4)
s = inputs.hemisphere(40, 60e-3)
op = dict(sigma=1e-4, v=1500.0, fs=40e6, n_samples=2048, t0=0.0, k=3.0)
KEYS = ("GPAIR_NO_TAB", "GPAIR_ADJ_NO_MP", "GPAIR_ADJ_NO_LCF", "GPAIR_ADJ_NO_T", "GPAIR_PIPELINE")
NM = {"GPAIR_ADJ_NO_MP": "1"}
for env in ({}, NM, dict(NM, GPAIR_ADJ_NO_LCF="1"), dict(NM, GPAIR_ADJ_NO_LCF="1", GPAIR_ADJ_NO_T="1"),
            {"GPAIR_NO_TAB": "1"}, dict(NM, GPAIR_NO_TAB="1"), {"GPAIR_PIPELINE": "1"}, dict(NM, GPAIR_PIPELINE="1"),
            {"GPAIR_PIPELINE": "1", "GPAIR_NO_TAB": "1"}):
    for key in KEYS:
        os.environ.pop(key, None)
    os.environ.update(env)
    info = run(c, s, op)
    print("path", env, "tab", info["tab"], "adj", info["adj_kernel"], flush=True)
for key in KEYS:
    os.environ.pop(key, None)
# the double-buffered cp.async forward and the moment-polynomial / LCF adjoints at other window lengths
for env in ({}, NM):
    os.environ.update(env)
    for W in (12, 24, 32):
        sw = W * (1500.0 / 40e6) / 6.0
        print("W", W, env, run(inputs.grid_centers(6, 6, 6, sw), s, dict(op, sigma=sw))["adj_kernel"], flush=True)
    for key in KEYS:
        os.environ.pop(key, None)
cfg1 = inputs.CONFIGS["cfg1"]
print("cfg1", run(cfg1.centers(), cfg1.sensors(), cfg1.op_kwargs())["adj_kernel"], flush=True)
print("assa (moment-polynomial adjoint)", run(c, s, op, assa=True)["adj_kernel"], flush=True)
os.environ["GPAIR_ADJ_NO_MP"] = "1"
print("assa (lane-per-kernel adjoint)", run(c, s, op, assa=True)["adj_kernel"], flush=True)
os.environ.pop("GPAIR_ADJ_NO_MP", None)
sig = np.full(c.shape[1], 1e-4, np.float32)
print("general", run(c, s, op, sigmas=T(sig))["general"], flush=True)
# near field: sensors inside the grid
s_in = np.ascontiguousarray(np.array([[0.0, 1e-4, -2e-4], [0.0, 0.0, 1e-4], [0.0, 3e-4, 0.0]], np.float32).T)
print("near", run(c, s_in, op, near_field=True)["near_pairs"], flush=True)
ctx = gpair.Context(T(c), T(s), sigma=1e-4, v=1500.0, fs=40e6, n_samples=2048)
gv = torch.empty(c.shape[1], device="cuda")
vv = torch.empty(1, device="cuda")
ctx.vcr(T(inputs.dense_amplitudes(c.shape[1])), (8, 8, 8), beta=0.5, eps=1e-8, grad=gv, value=vv)
torch.cuda.synchronize()
ctx.close()
print("done", flush=True)
