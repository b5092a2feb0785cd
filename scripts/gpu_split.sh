#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for S in 1 2 4 8; do
  GPAIR_FWD_SPLIT=$S timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('split $S', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['roofline']['kernel_ms'].items()})" >> gpurun_out/${T}_split.txt 2>&1
  GPAIR_FWD_SPLIT=$S timeout 600 python scripts/parity_report.py cfg4 cfg5 2>&1 | grep -A1 "\[" | grep forward >> gpurun_out/${T}_split.txt
done
GPAIR_FWD_SPLIT=4 GPAIR_FWD_CPR=8 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('split 4 cpr 8', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['roofline']['kernel_ms'].items()})" >> gpurun_out/${T}_split.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
cat gpurun_out/${T}_split.txt
