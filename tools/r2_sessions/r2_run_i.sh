#!/bin/bash
set -u
for sh in 0 1 2 3; do for a in "--kind constant" "--kind ramp"; do
  echo "== shape=$sh $a"; FGBD_LF_SHAPE=$sh timeout 120 python tools/profile_frame.py $a --frames 4 2>&1 | tail -1
done; done
for v in 13; do for a in "--kind constant" "--kind ramp" "--kind ramp --n 8000000"; do
  echo "== variant=$v $a"; FGBD_LF_VARIANT=$v timeout 120 python tools/profile_frame.py $a --frames 4 2>&1 | tail -1
done; done
