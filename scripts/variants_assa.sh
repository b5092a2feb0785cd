#!/bin/bash
# compile-time variants of the ASSA kernels, timed with bench --op assa (flags kept exported for the bench)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for V in "$@"; do
  export GPAIR_NVCC_FLAGS="$V"
  python paper_2602_03893_b200/build.py --force > /dev/null 2>&1 || { echo "build failed: $V"; continue; }
  R=$(timeout 600 python bench.py --op assa --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1)
  echo "VARIANT [$V] $(echo $R | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), {k: round(v,2) for k,v in d["roofline"]["kernel_ms"].items()})')"
done
