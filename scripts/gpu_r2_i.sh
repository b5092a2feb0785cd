#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for L in libgpair.so libgpair_x2.so libgpair_x3.so; do
  GPAIR_LIB=$L timeout 600 python scripts/parity_report.py cfg5 2>&1 | grep -B1 forward >> gpurun_out/r2i.txt
done
GPAIR_FWD_SPLIT=8 GPAIR_FWD_CPR=2 timeout 600 python scripts/parity_report.py cfg5 2>&1 | grep -B1 forward >> gpurun_out/r2i.txt
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r2i_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2i_pytest.log
cat gpurun_out/r2i.txt
