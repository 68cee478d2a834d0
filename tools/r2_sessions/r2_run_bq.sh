#!/bin/bash
# Round 2 session BQ: decide-before-sweep as its own instantiation, chosen
# per context from the last scan's outcome (FGBD_LF_HOLD -1 auto / 0 / 1).
set -u
O=gpurun_out/r2bq; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fuzz_gpu.py tests/test_concurrency_gpu.py tests/test_reuse.py -m gpu -x -q -p no:cacheprovider > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
for rep in 1 2; do
for h in -1 0 1; do
  for k in ramp two-tone constant; do
    echo "== hold=$h $k"; FGBD_LF_HOLD=$h timeout 120 python tools/profile_frame.py --kind $k --frames 4 2>&1 | tail -1
  done
done
done
