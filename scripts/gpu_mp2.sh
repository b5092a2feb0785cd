#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -s -k "full_size or random_suite or cfg1" --timeout 600 > gpurun_out/pytest_mp_s.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_mp_s.log
CFG=cfg4 K=k_adjoint_mp TAG=mp1 KEEP=1 bash scripts/gpu_ncu1.sh
grep -E "adjoint cols|forward rows" gpurun_out/pytest_mp_s.log | head -20
cat gpurun_out/prof_cfg4_k_adjoint_mp_mp1_summary.txt | head -40
