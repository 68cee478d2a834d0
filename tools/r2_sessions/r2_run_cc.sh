#!/bin/bash
# Round 2 session CC: the three channels' Jacobi on three host threads
# (FGBD_JACOBI_THREADS) -- tests, A/B, host timeline, bench.
set -u
O=gpurun_out/r2cc; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/tests.log 2>&1; echo "tests rc=$?"; tail -1 $O/tests.log
timeout 300 python tools/concurrency_repro.py | tail -1
for rep in 1 2; do
for m in 1 0; do
  for k in ramp two-tone; do
    echo "== threads=$m $k"; FGBD_JACOBI_THREADS=$m timeout 120 python tools/profile_frame.py --kind $k --frames 4 2>&1 | tail -1
  done
done
done
for m in 1 0; do FGBD_JACOBI_THREADS=$m FGBD_HOST_TLOG=1 timeout 120 python tools/host_overhead.py 2>&1 | grep "host tlog" | tail -2; done
for m in 1 0; do
FGBD_JACOBI_THREADS=$m python bench.py --no-cpu-baseline --no-e2e > $O/bench_$m.json 2> $O/bench_$m.err; python -c "import json; d=json.loads(open('$O/bench_$m.json').read().strip().splitlines()[-1]); print('threads=$m ramp', round(d['value'],1), d['stage_ms'])"
FGBD_JACOBI_THREADS=$m python bench.py --kind two-tone --no-cpu-baseline --no-e2e > $O/bench_tt_$m.json 2> $O/bench_tt_$m.err; python -c "import json; d=json.loads(open('$O/bench_tt_$m.json').read().strip().splitlines()[-1]); print('threads=$m two-tone', round(d['value'],1))"
done
