#!/bin/bash
# tests of the adjoint paths + 3 repeated cfg4 benches (adjoint ms)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py tests/test_gpu_assa.py -q -x --timeout 900 > gpurun_out/pytest_ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab.log
tail -2 gpurun_out/pytest_ab.log
for r in 1 2 3; do
  timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), {k: round(v,3) for k,v in d['roofline']['kernel_ms'].items()})"
done
