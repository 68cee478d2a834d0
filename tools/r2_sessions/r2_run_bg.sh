#!/bin/bash
# Round 2 session BG: graph parity with the current k_slg; full ncu captures
# of k_rows and k_noise2 (ramp and constant).
set -u
O=gpurun_out/r2bg; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_large_frames.py tests/test_slab_fuzz.py tests/test_fuzz_gpu.py tests/test_frame_8m.py -m gpu -x -q -p no:cacheprovider > $O/tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/tests.log
for k in ramp constant; do
ncu --set full --clock-control none --import-source on -k regex:"k_rows|k_noise2" --launch-skip 2 --launch-count 2 -o $O/side_$k python tools/profile_frame.py --kind $k --frames 2 > $O/ncu_$k.log 2>&1; echo "ncu $k rc=$?"
done
