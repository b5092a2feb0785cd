#!/bin/bash
# fp32 tail accumulation in k_adjoint_mp (GPAIR_MP_TAILF32): parity values at every config + A/B timing
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python paper_2602_03893_b200/build.py --force > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -s -q -x --timeout 900 > gpurun_out/pytest_parity_values_tailf32.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_parity_values_tailf32.log
bash scripts/gpu_ab_adj.sh
bash scripts/variants.sh "-DGPAIR_MP_TAILF32=0" "" "-DGPAIR_MP_TAILF32=0" "" > gpurun_out/variants_tailf32.txt 2>&1
cat gpurun_out/variants_tailf32.txt
