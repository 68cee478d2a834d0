#!/bin/bash
# Round 2 session BB: slg.cu with batched loads -- graph parity + timings.
set -u
O=gpurun_out/r2bb; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_large_frames.py tests/test_slab_fuzz.py tests/test_fuzz_gpu.py -m gpu -x -q -p no:cacheprovider > $O/tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/tests.log
for coop in 1 0; do
  for k in ramp two-tone constant; do
    echo "== coop=$coop $k"; FGBD_SLG_COOP=$coop timeout 120 python tools/profile_frame.py --kind $k --frames 4 2>&1 | tail -1
    echo "== coop=$coop $k shuffled"; FGBD_SLG_COOP=$coop timeout 120 python tools/profile_frame.py --kind $k --order shuffle --frames 4 2>&1 | tail -1
  done
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_ramp.csv python tools/profile_frame.py --frames 3 > $O/ncu_l.log 2>&1; echo "launches rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_shuffled.csv python tools/profile_frame.py --kind constant --order shuffle --frames 3 > $O/ncu_l2.log 2>&1; echo "launches2 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_slg --launch-skip 2 --launch-count 1 -o $O/slg_ramp python tools/profile_frame.py --frames 3 > $O/ncu_f.log 2>&1; echo "ncu full rc=$?"
