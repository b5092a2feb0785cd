#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r2p_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2p_pytest.log
timeout 1500 python scripts/ir_runs.py > gpurun_out/r2p_ir.log 2>&1
echo "ir rc=$?" >> gpurun_out/r2p_ir.log
bash scripts/gpu_sanitize.sh > gpurun_out/r2p_sanitize.log 2>&1
tail -3 gpurun_out/r2p_pytest.log; cat gpurun_out/r2p_ir.log; cat gpurun_out/r2p_sanitize.log
