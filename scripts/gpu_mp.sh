#!/bin/bash
# Moment-polynomial adjoint: paths + full-size parity + a short bench.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py -q --timeout 900 ${PYTEST_ARGS} > gpurun_out/pytest_mp.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_mp.log
timeout 600 python bench.py --steps 10 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench_mp.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_mp.log
tail -30 gpurun_out/pytest_mp.log; tail -c 2500 gpurun_out/bench_mp.log
