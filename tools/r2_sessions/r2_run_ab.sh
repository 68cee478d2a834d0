#!/bin/bash
# A/B of the filter against the r2q library on one box (3 alternations).
set -u
for rep in 1 2 3; do
for lib in paper_2401_09721_b200/_lib/libfgbd_b200.so tools/_lib_r2q.so; do
  for a in "--kind ramp" "--kind two-tone"; do
    echo "== lib=$lib $a"; FGBD_LIB_PATH=$lib timeout 120 python tools/profile_frame.py $a --frames 4 2>&1 | tail -1
  done
done
done
