#!/bin/bash
# A/B of the factorised-Gaussian (TAB) path vs the per-sample MUFU path: parity + times.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python scripts/parity_report.py ${CFGS:-cfg1 cfg2 cfg4} > gpurun_out/tab_on.log 2>&1
GPAIR_NO_TAB=1 timeout 600 python scripts/parity_report.py ${CFGS:-cfg1 cfg2 cfg4} > gpurun_out/tab_off.log 2>&1
if [ -n "$TESTS" ]; then timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log; fi
cat gpurun_out/tab_on.log gpurun_out/tab_off.log | tail -20
