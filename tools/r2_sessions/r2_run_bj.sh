#!/bin/bash
# Round 2 session BJ: k_noise2 occupancy sweep (FGBD_NE_MINB 4/5/6/7) and
# the k_rows grid (8 blocks/SM grid-stride vs one row per thread).
set -u
for rep in 1 2; do
for lib in paper_2401_09721_b200/_lib/libfgbd_b200.so tools/_lib_ne4.so tools/_lib_ne5.so tools/_lib_ne7.so; do
  for k in ramp constant; do
    echo "== lib=$lib $k"; FGBD_LIB_PATH=$lib timeout 120 python tools/profile_frame.py --kind $k --frames 4 2>&1 | tail -1
  done
done
for k in ramp constant; do
  echo "== rows_grid=1 $k"; FGBD_ROWS_GRID=1 timeout 120 python tools/profile_frame.py --kind $k --frames 4 2>&1 | tail -1
done
done
