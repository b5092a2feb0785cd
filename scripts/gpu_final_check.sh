#!/bin/bash
# the whole -m gpu suite + smoke + cfg4 exact and ASSA bench lines at HEAD
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_${TAG}.log
tail -2 gpurun_out/pytest_gpu_${TAG}.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_${TAG}.log
tail -2 gpurun_out/smoke_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_${TAG}.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --op assa --no-cpu-baseline > gpurun_out/bench_assa_${TAG}.log 2>&1; echo "bench assa rc=$?"
tail -1 gpurun_out/bench_${TAG}.log | cut -c1-400
tail -1 gpurun_out/bench_assa_${TAG}.log | cut -c1-400
