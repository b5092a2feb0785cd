#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for V in "libgpair.so 1" "libgpair.so 0" "libgpair_u2.so 1"; do set -- $V
  echo "== $1 union $2" >> gpurun_out/${T}.txt
  GPAIR_FWD_UNION=$2 GPAIR_LIB=$1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['roofline']['kernel_ms'].items()})" >> gpurun_out/${T}.txt 2>&1
  GPAIR_FWD_UNION=$2 GPAIR_LIB=$1 timeout 600 python scripts/parity_report.py cfg1 cfg2 cfg4 2>&1 | grep forward >> gpurun_out/${T}.txt
done
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
cat gpurun_out/${T}.txt; tail -2 gpurun_out/${T}_pytest.log
