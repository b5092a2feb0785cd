#!/bin/bash
# parity only, several libs: LIBS=... CFGS=... T=tag
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for L in $LIBS; do
  GPAIR_LIB=$L timeout 600 python scripts/parity_report.py $CFGS >> gpurun_out/${T}_par.txt 2>&1
done
cat gpurun_out/${T}_par.txt
