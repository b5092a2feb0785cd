#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for L in libgpair.so libgpair_p1.so libgpair_p1m6.so; do for A in 8 4 2; do
  echo "== $L adj cpr $A" >> gpurun_out/${T}.txt
  GPAIR_ADJ_CPR=$A GPAIR_LIB=$L timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['roofline']['kernel_ms'].items()}, d['config']['layout'])" >> gpurun_out/${T}.txt 2>&1
done; done
cat gpurun_out/${T}.txt
