#!/bin/bash
# bench + parity for several library builds: LIBS="libgpair_va.so ..." T=tag
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for L in $LIBS; do
  GPAIR_LIB=$L timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['roofline']['kernel_ms'].items()})" >> gpurun_out/${T}_libs.txt 2>&1
  [ -n "$PARITY" ] && GPAIR_LIB=$L timeout 600 python scripts/parity_report.py $PARITY >> gpurun_out/${T}_libs.txt 2>&1
done
cat gpurun_out/${T}_libs.txt
