#!/bin/bash
# Round 2 session BM: filter launched before the host NE finish (sigma_est
# through mapped memory, FGBD_EARLY_LF): parity, A/B, host timeline.
set -u
O=gpurun_out/r2bm; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/tests.log
for rep in 1 2; do
for e in 1 0; do
  for k in ramp two-tone constant; do
    echo "== early=$e $k"; FGBD_EARLY_LF=$e timeout 120 python tools/profile_frame.py --kind $k --frames 4 2>&1 | tail -1
  done
done
done
FGBD_HOST_TLOG=1 timeout 120 python tools/host_overhead.py 2>&1 | tail -4
python bench.py --no-cpu-baseline --no-e2e > $O/bench_frame.json 2> $O/bench_frame.err; echo "bench rc=$?"
python bench.py --kind two-tone --no-cpu-baseline --no-e2e > $O/bench_twotone.json 2> $O/bench_twotone.err; echo "bench2 rc=$?"
