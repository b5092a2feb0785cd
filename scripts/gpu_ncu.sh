#!/bin/bash
# ncu evidence: launch list of a short bench, and --set full on the top kernels.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CFG=${CFG:-cfg4}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${CFG}.csv \
    python bench.py --config $CFG --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_forward|k_adjoint" -c 3 \
    -o gpurun_out/prof_${CFG} python scripts/profile_once.py $CFG > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
tail -3 gpurun_out/ncu_full.log
