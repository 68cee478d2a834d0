#!/bin/bash
# Round 2 session BV: NE results posted to mapped host memory (FGBD_NE_MAIL)
# -- full GPU suite, A/B, host timeline, bench.
set -u
O=gpurun_out/r2bv; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
for rep in 1 2; do
for m in 1 0; do
  for k in ramp two-tone constant; do
    echo "== mail=$m $k"; FGBD_NE_MAIL=$m timeout 120 python tools/profile_frame.py --kind $k --frames 4 2>&1 | tail -1
  done
done
done
FGBD_HOST_TLOG=1 timeout 120 python tools/host_overhead.py > $O/ho.log 2>&1; grep "host tlog" $O/ho.log | tail -2; tail -2 $O/ho.log
for rep in 1 2; do
python bench.py --no-cpu-baseline > $O/bench_$rep.json 2> $O/bench_$rep.err
python -c "import json; d=json.loads(open('$O/bench_$rep.json').read().strip().splitlines()[-1]); print('rep $rep', round(d['value'],1), d['ms_per_step'], d['stage_ms'], d['e2e']['value'], d['e2e_pageable']['value'])"
done
python bench.py --kind two-tone --no-cpu-baseline --no-e2e > $O/bench_tt.json 2> $O/bench_tt.err; python -c "import json; d=json.loads(open('$O/bench_tt.json').read().strip().splitlines()[-1]); print('two-tone', round(d['value'],1))"
python bench.py --workload video > $O/bench_video.json 2> $O/bench_video.err; python -c "import json; d=json.loads(open('$O/bench_video.json').read().strip().splitlines()[-1]); print('video', round(d['value'],1))"
