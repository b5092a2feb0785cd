#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_assa.py -q -s -x --timeout 600 > gpurun_out/pytest_assa_fwd.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_assa_fwd.log
grep -E "assa fwd|assa forward|passed|failed" gpurun_out/pytest_assa_fwd.log | tail -8
timeout 600 python bench.py --op assa --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_assa_fwd.log 2>&1
python -c "
import json
for l in open('gpurun_out/bench_assa_fwd.log'):
    if l.startswith('{'):
        d=json.loads(l); print(round(d['ms_per_step'],2), {k: round(v,3) for k,v in d['roofline']['kernel_ms'].items()})"
