#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for L in libgpair.so libgpair_f32s.so; do for S in 2 4; do
  echo "== $L split $S" >> gpurun_out/r2n.txt
  GPAIR_FWD_SPLIT=$S GPAIR_LIB=$L timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['roofline']['kernel_ms'].items()})" >> gpurun_out/r2n.txt 2>&1
  GPAIR_FWD_SPLIT=$S GPAIR_LIB=$L timeout 600 python scripts/parity_report.py cfg2 cfg4 cfg5 2>&1 | grep forward >> gpurun_out/r2n.txt
done; done
cat gpurun_out/r2n.txt
