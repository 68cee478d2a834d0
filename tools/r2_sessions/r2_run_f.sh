#!/bin/bash
# Round 2 session F: split-phase grid barrier A/B, k_prep grid A/B, parity.
set -u
O=gpurun_out/r2f; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/gpu_tests.log
for lib in paper_2401_09721_b200/_lib/libfgbd_b200.so tools/_lib_nosplit.so; do
  for a in "--kind ramp" "--kind constant" "--kind two-tone" "--kind ramp --n 8000000"; do
    echo "== lib=$lib $a"; FGBD_LIB_PATH=$lib timeout 120 python tools/profile_frame.py $a --frames 4 2>&1 | tail -1
  done
done
for pm in 2 4 8; do for a in "--kind ramp" "--kind constant"; do
  echo "== prep_mult=$pm $a"; FGBD_PREP_MULT=$pm timeout 120 python tools/profile_frame.py $a --frames 4 2>&1 | tail -1
done; done
echo done
