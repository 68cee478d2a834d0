#!/bin/bash
# One GPU session: parity tests, LF variant timings.  Usage: tools/gpu_round.sh [notests] [variants...]
mkdir -p gpurun_out
if [ "$1" != "notests" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
fi
shift
VARS=${@:-"0 2"}
for v in $VARS; do for p in 0 1; do
  echo "== variant=$v persist=$p"; FGBD_LF_VARIANT=$v FGBD_L2_PERSIST=$p timeout 120 python tools/profile_frame.py --frames 4 2>&1 | tail -1
done; done
for k in two-tone constant; do echo "== $k"; timeout 120 python tools/profile_frame.py --kind $k --frames 3 2>&1 | tail -1; done
