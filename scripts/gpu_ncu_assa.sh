#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-a1}
for K in k_assa_forward k_assa_adjoint; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -c 1 \
      -o gpurun_out/prof_cfg4_${K}_${TAG} -f python scripts/profile_once.py cfg4 assa > gpurun_out/ncu_full_${K}.log 2>&1
  echo "full $K rc=$?"
done
