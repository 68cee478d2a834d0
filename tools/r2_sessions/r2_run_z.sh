#!/bin/bash
set -u
O=gpurun_out/r2z; mkdir -p $O
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_constant.csv python tools/profile_frame.py --kind constant --frames 3 > $O/ncu_l.log 2>&1; echo "launches rc=$?"
