#!/bin/bash
# compute-sanitizer is closed on this pool: a bounds-checked variant of libgpair (GPAIR_MP_CHECK=1 traps
# on any out-of-range staged copy, table row or rare-path sample) runs the GPU tests of every
# moment-polynomial path; a trap fails the launch and the test.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export GPAIR_LIB=libgpair_check.so GPAIR_NVCC_FLAGS="-DGPAIR_MP_CHECK=1"
python paper_2602_03893_b200/build.py --force > gpurun_out/mp_check_build.log 2>&1 || { echo "build failed"; exit 1; }
grep -c "MP_CHECK\|trap" gpurun_out/mp_check_build.log > /dev/null
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_mp_check.log 2>&1
echo "pytest (GPAIR_MP_CHECK=1) rc=$?" >> gpurun_out/pytest_mp_check.log
tail -3 gpurun_out/pytest_mp_check.log
