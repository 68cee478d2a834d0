#!/bin/bash
set -u
for lib in paper_2401_09721_b200/_lib/libfgbd_b200.so tools/_lib_cg64.so tools/_lib_cg150.so tools/_lib_cg512.so tools/_lib_na512.so tools/_lib_ef512.so; do
  for a in "--kind ramp" "--kind constant" "--kind two-tone" "--kind ramp --order shuffle"; do
    echo "== lib=$lib $a"; FGBD_LIB_PATH=$lib timeout 120 python tools/profile_frame.py $a --frames 4 2>&1 | tail -1
  done
done
