#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_row32.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_row32.log
tail -3 gpurun_out/pytest_row32.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -s -k "full_size or cfg1" > gpurun_out/pytest_row32_s.log 2>&1
grep -E "adjoint" gpurun_out/pytest_row32_s.log
for V in 0 1; do
  GPAIR_MP_ROW48=$V timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_row48_$V.log 2>&1
  python -c "
import json
for l in open('gpurun_out/bench_row48_$V.log'):
    if l.startswith('{'):
        d=json.loads(l); print('ROW48=$V', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['roofline']['kernel_ms'].items()})"
done
