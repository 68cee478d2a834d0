#!/bin/bash
# Round 2 session BW: device-resident colours expanded by k_rows
# (FGBD_ROWS_EXPAND) -- full GPU suite, A/B, bench.
set -u
O=gpurun_out/r2bw; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
for rep in 1 2; do
for m in 1 0; do
  for k in ramp two-tone constant; do
    echo "== expand=$m $k"; FGBD_ROWS_EXPAND=$m timeout 120 python tools/profile_frame.py --kind $k --frames 4 2>&1 | tail -1
  done
done
done
for m in 1 0; do
for rep in 1 2; do
FGBD_ROWS_EXPAND=$m python bench.py --no-cpu-baseline --no-e2e > $O/bench_${m}_$rep.json 2> $O/bench_${m}_$rep.err
python -c "import json; d=json.loads(open('$O/bench_${m}_$rep.json').read().strip().splitlines()[-1]); print('expand=$m rep $rep', round(d['value'],1), d['ms_per_step'], d['stage_ms'])"
done
done
FGBD_ROWS_EXPAND=1 python bench.py --kind two-tone --no-cpu-baseline --no-e2e > $O/bench_tt.json 2> $O/bench_tt.err; python -c "import json; d=json.loads(open('$O/bench_tt.json').read().strip().splitlines()[-1]); print('two-tone', round(d['value'],1))"
