#!/bin/bash
# Round 2 session BF: full ncu capture of k_slg (ramp, sorted input).
set -u
O=gpurun_out/r2bf; mkdir -p $O
ncu --set full --clock-control none --import-source on -k regex:k_slg --launch-skip 1 --launch-count 1 -o $O/slg_ramp python tools/profile_frame.py --frames 2 > $O/ncu_f.log 2>&1; echo "ncu full rc=$?"
