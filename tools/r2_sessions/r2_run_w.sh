#!/bin/bash
set -u
for lib in paper_2401_09721_b200/_lib/libfgbd_b200.so tools/_lib_farcg512.so tools/_lib_farcg4096.so; do
  for a in "--kind ramp" "--kind constant" "--kind ramp --n 8000000"; do
    echo "== lib=$lib $a"; FGBD_LIB_PATH=$lib timeout 120 python tools/profile_frame.py $a --frames 4 2>&1 | tail -1
  done
done
