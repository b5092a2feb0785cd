#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_assa.py tests/test_gpu_paths.py -q -s -x --timeout 600 > gpurun_out/pytest_assa_mp.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_assa_mp.log
grep -E "assa adjoint|cfg4|passed|failed|Error|error" gpurun_out/pytest_assa_mp.log | head -40
timeout 600 python bench.py --op assa --steps 10 --warmup 3 > gpurun_out/bench_assa_mp.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_assa_mp.log
python - <<'P'
import json
for l in open("gpurun_out/bench_assa_mp.log"):
    if l.startswith("{"):
        d=json.loads(l); print("ms/step", d["ms_per_step"], d["roofline"]["kernel_ms"])
P
tail -2 gpurun_out/bench_assa_mp.log | cut -c1-300
