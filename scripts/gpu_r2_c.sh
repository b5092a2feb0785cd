#!/bin/bash
# Round 2: fp64-chain LCF adjoint -- parity at SURVEY 8c sizes, timing, info
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python scripts/parity_report.py cfg1 cfg2 cfg4 cfg5 > gpurun_out/r2c_parity.txt 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2c_bench.txt 2>&1
python - >> gpurun_out/r2c_bench.txt 2>&1 <<'PY'
import torch, numpy as np
from paper_2602_03893_b200 import gpair, inputs
for name in ("cfg2", "cfg4", "cfg5"):
    cfg = inputs.CONFIGS[name]
    ctx = gpair.Context(torch.from_numpy(cfg.centers()).cuda(), torch.from_numpy(cfg.sensors()).cuda(), sigma=cfg.sig,
                        v=cfg.v, fs=cfg.fs, n_samples=cfg.n_samples, t0=cfg.t0, k=cfg.k)
    print(name, ctx.info())
    ctx.close()
PY
timeout 1200 python -m pytest tests -m gpu -q -x -k "paths or parity or collective" > gpurun_out/r2c_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2c_pytest.log
tail -3 gpurun_out/r2c_pytest.log
