#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for C in 16 8 4; do
  echo "== assa cpr $C" >> gpurun_out/r2t.txt
  GPAIR_FWD_CPR=$C timeout 600 python bench.py --op assa --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['roofline']['kernel_ms'].items()})" >> gpurun_out/r2t.txt 2>&1
done
timeout 900 python -m pytest tests/test_gpu_assa.py -q > gpurun_out/r2t_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2t_pytest.log
cat gpurun_out/r2t.txt; tail -2 gpurun_out/r2t_pytest.log
