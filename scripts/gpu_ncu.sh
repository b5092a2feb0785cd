#!/bin/bash
# ncu evidence: launch list of a short bench, and --set full on the top kernels
# (one ncu invocation per kernel: later kernels of a multi-kernel capture came back NaN).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CFG=${CFG:-cfg4}
TAG=${TAG:-r1}
if [ -z "$SKIP_LAUNCH" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${CFG}.csv \
    python bench.py --config $CFG --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1
echo "launch list rc=$?"
fi
for K in k_forward k_adjoint; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -c 1 \
      -o gpurun_out/prof_${CFG}_${K}_${TAG} -f python scripts/profile_once.py $CFG > gpurun_out/ncu_full_${K}.log 2>&1
  echo "full $K rc=$?"
done
if [ -n "$PROFILE_REDUCE" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_reduce" -c 1 \
      -o gpurun_out/prof_${CFG}_k_reduce_${TAG} -f python scripts/profile_once.py $CFG > gpurun_out/ncu_full_k_reduce.log 2>&1
  echo "full k_reduce rc=$?"
fi
