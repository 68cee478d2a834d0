#!/bin/bash
# Round 2 session BU: 8M frame -- launch list and the k_slg phase timeline.
set -u
O=gpurun_out/r2bu; mkdir -p $O
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_8m.csv python tools/profile_frame.py --n 8000000 --frames 2 > $O/ncu_l.log 2>&1; echo "launches rc=$?"
FGBD_SLG_TLOG=1 timeout 200 python tools/profile_frame.py --n 8000000 --frames 2 2>&1 | grep -E "slg phase|frame" | tail -14
