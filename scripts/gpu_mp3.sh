#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py -q -s -x --timeout 600 > gpurun_out/pytest_fm1.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_fm1.log
grep -E "adjoint cols|passed|failed|Error|error" gpurun_out/pytest_fm1.log | head -20
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_fm1.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_fm1.log
python - <<'P'
import json
for l in open("gpurun_out/bench_fm1.log"):
    if l.startswith("{"):
        d=json.loads(l); print("ms/step", d["ms_per_step"], d["roofline"]["kernel_ms"])
P
tail -3 gpurun_out/bench_fm1.log | cut -c1-300
CFG=cfg4 K=k_forward_mp TAG=fm1 KEEP=1 bash scripts/gpu_ncu1.sh
head -32 gpurun_out/prof_cfg4_k_forward_mp_fm1_summary.txt; head -30 gpurun_out/prof_cfg4_k_forward_mp_fm1_sassmix.txt
