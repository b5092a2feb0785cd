#!/bin/bash
# Round 2, numerics experiment: exact fp64 pair values (x2: fp64 ToF, x3: fp32 ToF) vs the
# shipped kernels, and shorter forward accumulation chains (GPAIR_FWD_CPR).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for L in libgpair.so libgpair_x2.so libgpair_x3.so; do
  GPAIR_LIB=$L timeout 900 python scripts/parity_report.py cfg2 cfg4 >> gpurun_out/r2b_parity.txt 2>&1
done
for C in 8 4 2; do
  echo "GPAIR_FWD_CPR=$C" >> gpurun_out/r2b_parity.txt
  GPAIR_FWD_CPR=$C timeout 900 python scripts/parity_report.py cfg4 >> gpurun_out/r2b_parity.txt 2>&1
done
timeout 600 python -m pytest tests/test_gpu_collective.py "tests/test_gpu_parity.py::test_geometry_check_is_exact_per_pair" -q -s > gpurun_out/r2b_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2b_tests.log
tail -3 gpurun_out/r2b_tests.log
