#!/bin/bash
# compile-time stage index in k_adjoint_mp (GPAIR_MP_STAGE_UNROLL): path/parity/ASSA tests + A/B timing
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python paper_2602_03893_b200/build.py --force > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py tests/test_gpu_assa.py -q -x --timeout 900 > gpurun_out/pytest_unroll.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_unroll.log
tail -2 gpurun_out/pytest_unroll.log
bash scripts/variants.sh "" "-DGPAIR_MP_STAGE_UNROLL=0" "" "-DGPAIR_MP_STAGE_UNROLL=0" > gpurun_out/variants_unroll.txt 2>&1
cat gpurun_out/variants_unroll.txt
for V in "" "-DGPAIR_MP_STAGE_UNROLL=0"; do
  export GPAIR_NVCC_FLAGS="$V"
  python paper_2602_03893_b200/build.py --force > /dev/null 2>&1
  R=$(timeout 600 python bench.py --op assa --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1)
  echo "ASSA [$V] $(echo $R | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), {k: round(v,2) for k,v in d["roofline"]["kernel_ms"].items()})')" | tee -a gpurun_out/variants_unroll.txt
done
