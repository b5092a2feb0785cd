#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py tests/test_gpu_assa.py -q -x --timeout 900 > gpurun_out/pytest_slot.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_slot.log
tail -2 gpurun_out/pytest_slot.log
for V in 0 1; do
  GPAIR_MP_SLOT_RUNTIME=$V timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_slot_$V.log 2>&1
  python -c "
import json
for l in open('gpurun_out/bench_slot_$V.log'):
    if l.startswith('{'):
        d=json.loads(l); print('SLOT_RUNTIME=$V', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['roofline']['kernel_ms'].items()})"
done
