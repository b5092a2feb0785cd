#!/bin/bash
# one ncu --set full capture of kernel regex $K at config $CFG; summaries are written next to
# the report (scripts/ncu_summary.py, scripts/sass_mix.py) and the report itself is kept only
# with KEEP=1 (gpurun brings back <= 64 MiB)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CFG=${CFG:-cfg4}; K=${K:-k_adjoint}; TAG=${TAG:-x}
REP=gpurun_out/prof_${CFG}_${KN:-$K}_${TAG}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -c 1 \
    -o $REP -f python scripts/profile_once.py $CFG $ARGS > gpurun_out/ncu_full_${KN:-$K}_${TAG}.log 2>&1
echo "full $K rc=$?"
python scripts/ncu_summary.py $REP.ncu-rep > ${REP}_summary.txt 2>&1
python scripts/sass_mix.py $REP.ncu-rep ${UNITS:-268435456} > ${REP}_sassmix.txt 2>&1
[ -z "$KEEP" ] && rm -f $REP.ncu-rep
true
