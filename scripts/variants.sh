#!/bin/bash
# Build + bench several compile-time variants on the GPU box (forward tuning).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for V in "$@"; do
  # the flags stay exported for the bench too: build.build() keys its cache on them (a bench run
  # without them would silently rebuild the default library)
  export GPAIR_NVCC_FLAGS="$V"
  python paper_2602_03893_b200/build.py --force > /dev/null 2>&1 || { echo "build failed: $V"; continue; }
  grep -A3 "k_adjoint_mp<2, false>\|k_adjoint_mpILi2ELb0" paper_2602_03893_b200/build/libgpair/ptxas.log | grep -m1 registers
  R=$(timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1)
  echo "VARIANT [$V] $(echo $R | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), {k: round(v,2) for k,v in d["roofline"]["kernel_ms"].items()})')"
done
