import sys, numpy as np
sys.path.insert(0, '.')
import oracle
from paper_2602_03893_b200 import inputs
f32 = np.float32
cfg = inputs.CONFIGS['cfg1']
c, s, op = cfg.centers(), cfg.sensors(), cfg.op_kwargs()
x = inputs.dense_amplitudes(cfg.M)
y_ref = oracle.forward(c, x, s, **op)
M, Nd, Nt = c.shape[1], s.shape[1], cfg.n_samples
v, fs, sig, ks = cfg.v, cfg.fs, cfg.sig, 3*cfg.sig
h = v/fs
# exact terms in fp64, vs variants
c64 = c.astype(np.float64); s64 = s.astype(np.float64)
r = np.sqrt(((c64[:, :, None] - s64[:, None, :])**2).sum(0))  # M x Nd
def metric(y):
    big = np.abs(y_ref) >= 1e-3*np.abs(y_ref).max()
    return np.linalg.norm(y-y_ref)/np.linalg.norm(y_ref), np.max(np.abs(y[big]-y_ref[big])/np.abs(y_ref[big]))
tn = np.arange(Nt)/fs
def accumulate(term_fn, dtype=np.float64):
    y = np.zeros((Nd, Nt), dtype)
    for i in range(M):
        d = r[i][:, None] - v*tn[None, :]
        mask = np.abs(d) < ks
        vals = term_fn(i, d, mask)
        y += np.where(mask, vals, 0).astype(dtype)
    return y
# 1) exact fp64 terms, fp64 accumulation (should be ~0)
print('fp64 terms', metric(accumulate(lambda i,d,m: x[i]*d*np.exp(-d*d/(2*sig*sig))/(2*r[i][:,None]))))
# 2) exact terms rounded to fp32, fp32 sequential accumulation
print('fp32-rounded terms, fp32 acc', metric(accumulate(lambda i,d,m: (x[i]*d*np.exp(-d*d/(2*sig*sig))/(2*r[i][:,None])).astype(f32), np.float32)))
# 3) d perturbed by 1e-11 m random
rng=np.random.default_rng(0)
for dd in [1e-11, 3e-11, 1e-10]:
    print('d err', dd, metric(accumulate(lambda i,d,m: x[i]*(d+dd*rng.standard_normal(d.shape[0])[:,None])*np.exp(-(d+dd*rng.standard_normal(d.shape[0])[:,None])**2/(2*sig*sig))/(2*r[i][:,None]))))
# 4) relative per-term error
for rel in [1e-7, 3e-7, 1e-6]:
    print('term rel err', rel, metric(accumulate(lambda i,d,m: x[i]*d*np.exp(-d*d/(2*sig*sig))/(2*r[i][:,None])*(1+rel*rng.standard_normal(d.shape)))))
