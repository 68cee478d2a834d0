# Compile-time filter variants (tools/_lib_*.so built by _build.build(defines=...)),
# A/B against the default library on one box, two alternating rounds.
run() { env "$@" python bench.py --no-cpu-baseline --no-e2e --steps 30 --warmup 5 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['stage_ms']
print('$*'.replace('FGBD_LIB_PATH=tools/_lib_',''), round(d['value'],1), round(d['roofline']['frac'],4), round(s['low_pass_filter_ms'],4))"; }
for r in 1 2; do
  run X=base
  for v in ${VARIANTS:-FGBD_ELL_POLICY2 FGBD_LF_PFD1 FGBD_LF_PFD4 FGBD_LF_ELLSMEM0 FGBD_LF_ELLSMEM2 FGBD_LF_PF0}; do
    run FGBD_LIB_PATH=tools/_lib_$v.so
  done
done
