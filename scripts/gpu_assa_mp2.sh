#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_assa.py -q -s -x --timeout 600 > gpurun_out/pytest_assa_mp.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_assa_mp.log
grep -E "assa adjoint|cfg4|passed|failed|Error|error" gpurun_out/pytest_assa_mp.log | head -40
CFG=cfg4 K=k_adjoint_mp ARGS=assa TAG=assa1 KEEP=1 bash scripts/gpu_ncu1.sh
head -32 gpurun_out/prof_cfg4_k_adjoint_mp_assa1_summary.txt; head -30 gpurun_out/prof_cfg4_k_adjoint_mp_assa1_sassmix.txt
