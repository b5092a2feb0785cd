#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_paths.py -q -s -x --timeout 900 -k "cluster or each_path" > gpurun_out/pytest_cluster.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cluster.log
grep -E "cluster|passed|failed|Error" gpurun_out/pytest_cluster.log | head -20
for CL in 1 2 4 8; do
  GPAIR_FWD_CLUSTER=$CL timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cluster_$CL.log 2>&1
  python -c "
import json
for l in open('gpurun_out/bench_cluster_$CL.log'):
    if l.startswith('{'):
        d=json.loads(l); print('CLUSTER=$CL', round(d['ms_per_step'],2), {k: round(v,3) for k,v in d['roofline']['kernel_ms'].items()})" || tail -5 gpurun_out/bench_cluster_$CL.log
done
