#!/bin/bash
# Round 2 session CA: k_lf_run as one 768-thread block per SM (FGBD_LF_SHAPE=4) vs 3 x 256.
set -u
for rep in 1 2; do
for sh in 0 4; do
  for k in ramp constant; do
    echo "== shape=$sh $k"; FGBD_LF_SHAPE=$sh timeout 120 python tools/profile_frame.py --kind $k --frames 4 2>&1 | tail -1
  done
  echo "== shape=$sh 8M"; FGBD_LF_SHAPE=$sh timeout 200 python tools/profile_frame.py --n 8000000 --frames 3 2>&1 | tail -1
done
done
