#!/bin/bash
# Round evidence on one B200: GPU tests, smoke, bench (JSON line), ncu launch
# list of a short bench, and one ncu --set full capture per hot kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-ev}
CFG=${CFG:-cfg4}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu_${TAG}.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_${TAG}.log
timeout 900 python bench.py --config $CFG > gpurun_out/bench_${TAG}.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_${TAG}.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${CFG}_${TAG}.csv \
    python bench.py --config $CFG --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_${TAG}.log 2>&1
echo "launch list rc=$?"
for K in k_forward k_adjoint_mp "k_reduce\$"; do
  KN=$(echo "$K" | tr -d '$\\')
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -c 1 \
      -o gpurun_out/prof_${CFG}_${KN}_${TAG} -f python scripts/profile_once.py $CFG > gpurun_out/ncu_full_${KN}_${TAG}.log 2>&1
  echo "full $KN rc=$?"
  python scripts/ncu_summary.py gpurun_out/prof_${CFG}_${KN}_${TAG}.ncu-rep > gpurun_out/ncu_summary_${KN}_${TAG}.txt 2>&1
  python scripts/sass_mix.py gpurun_out/prof_${CFG}_${KN}_${TAG}.ncu-rep 268435456 > gpurun_out/ncu_sassmix_${KN}_${TAG}.txt 2>&1
  [ -z "$KEEP_REP" ] && rm -f gpurun_out/prof_${CFG}_${KN}_${TAG}.ncu-rep
done
# the ASSA adjoint on the moment-polynomial kernel
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_adjoint_mp -c 1 \
    -o gpurun_out/prof_${CFG}_assa_k_adjoint_mp_${TAG} -f python scripts/profile_once.py $CFG assa > gpurun_out/ncu_full_assa_mp_${TAG}.log 2>&1
python scripts/ncu_summary.py gpurun_out/prof_${CFG}_assa_k_adjoint_mp_${TAG}.ncu-rep > gpurun_out/ncu_summary_assa_k_adjoint_mp_${TAG}.txt 2>&1
python scripts/sass_mix.py gpurun_out/prof_${CFG}_assa_k_adjoint_mp_${TAG}.ncu-rep 268435456 > gpurun_out/ncu_sassmix_assa_k_adjoint_mp_${TAG}.txt 2>&1
[ -z "$KEEP_REP" ] && rm -f gpurun_out/prof_${CFG}_assa_k_adjoint_mp_${TAG}.ncu-rep
# the ASSA forward
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_assa_forward -c 1 \
    -o gpurun_out/prof_${CFG}_k_assa_forward_${TAG} -f python scripts/profile_once.py $CFG assa > gpurun_out/ncu_full_assa_fwd_${TAG}.log 2>&1
python scripts/ncu_summary.py gpurun_out/prof_${CFG}_k_assa_forward_${TAG}.ncu-rep > gpurun_out/ncu_summary_k_assa_forward_${TAG}.txt 2>&1
python scripts/sass_mix.py gpurun_out/prof_${CFG}_k_assa_forward_${TAG}.ncu-rep 268435456 > gpurun_out/ncu_sassmix_k_assa_forward_${TAG}.txt 2>&1
[ -z "$KEEP_REP" ] && rm -f gpurun_out/prof_${CFG}_k_assa_forward_${TAG}.ncu-rep
# the other bench lines: the reference arm (fp64 oracle), the ASSA operator, cfg5 / cfg3
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_${TAG}.log 2>&1
timeout 600 python bench.py --op assa --no-cpu-baseline > gpurun_out/bench_assa_${TAG}.log 2>&1
for C in cfg5 cfg3; do timeout 600 python bench.py --config $C --no-cpu-baseline > gpurun_out/bench_${C}_${TAG}.log 2>&1; done
# NVTX: the library's stage ranges (domain "gpair") around each launch of one cfg1 iterate
timeout 300 ncu --nvtx --print-summary per-nvtx --metrics gpu__time_duration.sum --clock-control none \
    python scripts/profile_once.py cfg1 > gpurun_out/ncu_nvtx_${TAG}.txt 2>&1
tail -2 gpurun_out/pytest_gpu_${TAG}.log; tail -2 gpurun_out/smoke_${TAG}.log; tail -c 600 gpurun_out/bench_${TAG}.log
