#!/bin/bash
# one ncu --set full capture of kernel regex $K at config $CFG (default: the TAB adjoint at cfg4)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CFG=${CFG:-cfg4}; K=${K:-k_adjoint}; TAG=${TAG:-x}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -c 1 \
    -o gpurun_out/prof_${CFG}_${KN:-$K}_${TAG} -f python scripts/profile_once.py $CFG > gpurun_out/ncu_full_${KN:-$K}_${TAG}.log 2>&1
echo "full $K rc=$?"
