#!/bin/bash
# Round 2 session BI: occupancy variants of k_rows / k_noise2 (A/B, 2 reps),
# then the multi-channel host Jacobi's parity tests.
set -u
O=gpurun_out/r2bi; mkdir -p $O
for rep in 1 2; do
for lib in paper_2401_09721_b200/_lib/libfgbd_b200.so tools/_lib_rows4.so tools/_lib_ne8.so tools/_lib_both.so; do
  for k in ramp two-tone constant; do
    echo "== lib=$lib $k"; FGBD_LIB_PATH=$lib timeout 120 python tools/profile_frame.py --kind $k --frames 4 2>&1 | tail -1
  done
done
done
for lib in paper_2401_09721_b200/_lib/libfgbd_b200.so tools/_lib_both.so; do
FGBD_LIB_PATH=$lib ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$(basename $lib .so).csv python tools/profile_frame.py --frames 3 > $O/ncu_l.log 2>&1; echo "launches rc=$?"
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fuzz_gpu.py tests/test_device_finish.py tests/test_boundary.py -m gpu -x -q -p no:cacheprovider > $O/tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/tests.log
