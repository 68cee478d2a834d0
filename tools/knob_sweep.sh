run() { env "$@" python bench.py --no-cpu-baseline --no-e2e --steps 30 --warmup 5 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['stage_ms']
print('$*', round(d['value'],1), round(d['roofline']['frac'],4), {k:round(v,4) for k,v in s.items()})"; }
run X=0
run FGBD_LF_SHAPE=1
run FGBD_LF_SHAPE=2
run FGBD_LF_SHAPE=3
run FGBD_PREP_MULT=2
run FGBD_PREP_MULT=4
run FGBD_PREP_MULT=16
run FGBD_L2_PERSIST=1
run FGBD_LF_VARIANT=13
run X=1
