#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every kernel path (tiny instances)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "from paper_2602_03893_b200 import build as b; b.build()"
for T in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $T --error-exitcode 9 python scripts/sanitize_small.py > gpurun_out/sanitize_$T.log 2>&1
  echo "$T rc=$?"; tail -4 gpurun_out/sanitize_$T.log
done
