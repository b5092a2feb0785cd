cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -c "from paper_2602_03893_b200 import build; build.build()"
for r in 1 2 3; do for V in 0 1; do
  GPAIR_MP_SLOT_RUNTIME=$V timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('SLOT_RUNTIME=$V', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['roofline']['kernel_ms'].items()})"
done; done
