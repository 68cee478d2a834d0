#!/bin/bash
# Round 2 session BO: split first steps, k_fold2 as one wave (3 or 2 blocks/SM) vs off.
set -u
O=gpurun_out/r2bo; mkdir -p $O
for rep in 1 2; do
for v in "1 paper_2401_09721_b200/_lib/libfgbd_b200.so" "1 tools/_lib_f2m2.so" "0 paper_2401_09721_b200/_lib/libfgbd_b200.so"; do
  set -- $v
  for k in ramp two-tone constant; do
    echo "== early=$1 lib=$2 $k"; FGBD_EARLY_LF=$1 FGBD_LIB_PATH=$2 timeout 120 python tools/profile_frame.py --kind $k --frames 4 2>&1 | tail -1
  done
done
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_ramp.csv python tools/profile_frame.py --frames 3 > $O/ncu_l.log 2>&1; echo "launches rc=$?"
