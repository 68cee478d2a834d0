#!/bin/bash
# Round 2 session BN: split first steps -- per-kernel times and host timeline.
set -u
O=gpurun_out/r2bn; mkdir -p $O
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_ramp.csv python tools/profile_frame.py --frames 3 > $O/ncu_l.log 2>&1; echo "launches rc=$?"
FGBD_HOST_TLOG=1 timeout 120 python tools/host_overhead.py > $O/ho.log 2>&1; grep "host tlog" $O/ho.log | tail -3
FGBD_HOST_TLOG=1 FGBD_EARLY_LF=0 timeout 120 python tools/host_overhead.py > $O/ho0.log 2>&1; grep "host tlog" $O/ho0.log | tail -2
