#!/bin/bash
set -u
O=gpurun_out/r2p; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -4 $O/gpu_tests.log
for f in 1 0; do for a in "--kind ramp" "--kind two-tone" "--kind constant"; do
  echo "== fold=$f $a"; FGBD_MASK_FOLD=$f timeout 120 python tools/profile_frame.py $a --frames 4 2>&1 | tail -1
done; done
