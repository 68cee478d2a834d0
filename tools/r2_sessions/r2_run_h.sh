#!/bin/bash
set -u
for lib in paper_2401_09721_b200/_lib/libfgbd_b200.so tools/_lib_rcpdiv.so; do
  for a in "--kind ramp" "--kind constant" "--kind two-tone" "--kind ramp --n 8000000"; do
    echo "== lib=$lib $a"; FGBD_LIB_PATH=$lib timeout 120 python tools/profile_frame.py $a --frames 4 2>&1 | tail -1
  done
done
FGBD_LIB_PATH=tools/_lib_rcpdiv.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fuzz_gpu.py -q -p no:cacheprovider -x > gpurun_out/r2h_parity.log 2>&1; echo "parity(rcpdiv) rc=$?"; tail -2 gpurun_out/r2h_parity.log
