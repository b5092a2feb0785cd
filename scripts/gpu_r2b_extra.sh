#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CFG=cfg4 K=k_forward TAG=r2bsrc KEEP=1 bash scripts/gpu_ncu1.sh
timeout 1500 python scripts/ir_runs.py > gpurun_out/ir_runs_r2b.log 2>&1
echo "rc=$?" >> gpurun_out/ir_runs_r2b.log
cat gpurun_out/ir_runs_r2b.log | tail -5
