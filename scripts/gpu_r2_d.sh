#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${T:-r2d}
timeout 900 python scripts/parity_report.py cfg2 cfg4 > gpurun_out/${T}_parity.txt 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -k "paths or parity or collective or general or assa" > gpurun_out/${T}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
if [ -n "$NCU" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$NCU" -c 1 \
    -o gpurun_out/prof_cfg4_${NCU}_${T} -f python scripts/profile_once.py cfg4 > gpurun_out/ncu_${T}.log 2>&1
fi
tail -2 gpurun_out/${T}_pytest.log
