#!/bin/bash
# Round 2 session BH: k_rows / k_noise2 load hoisting + weight table: parity
# and an A/B against the previous commit's library.
set -u
O=gpurun_out/r2bh; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fuzz_gpu.py tests/test_reuse.py -m gpu -x -q -p no:cacheprovider > $O/tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/tests.log
for rep in 1 2 3; do
for lib in paper_2401_09721_b200/_lib/libfgbd_b200.so tools/_lib_head.so; do
  for k in ramp two-tone constant; do
    echo "== lib=$lib $k"; FGBD_LIB_PATH=$lib timeout 120 python tools/profile_frame.py --kind $k --frames 4 2>&1 | tail -1
  done
done
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_ramp.csv python tools/profile_frame.py --frames 3 > $O/ncu_l.log 2>&1; echo "launches rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_constant.csv python tools/profile_frame.py --kind constant --frames 3 > $O/ncu_l2.log 2>&1; echo "launches2 rc=$?"
