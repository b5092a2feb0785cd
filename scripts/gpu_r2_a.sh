#!/bin/bash
# Round 2, first GPU call: adjoint accumulation variants at SURVEY 8c sample sizes,
# the collective-path tests, then the whole GPU suite.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_gpu.txt
for L in libgpair_a0e0.so libgpair.so libgpair_a1e1.so libgpair_a0e1.so; do
  GPAIR_LIB=$L timeout 900 python scripts/parity_report.py cfg2 cfg4 cfg5 >> gpurun_out/r2a_parity.txt 2>&1
done
timeout 600 python -m pytest tests/test_gpu_collective.py -x -q -s > gpurun_out/r2a_collective.log 2>&1
echo "collective rc=$?" >> gpurun_out/r2a_collective.log
timeout 1800 python -m pytest tests -m gpu -q -s > gpurun_out/r2a_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2a_pytest_gpu.log
tail -5 gpurun_out/r2a_parity.txt
