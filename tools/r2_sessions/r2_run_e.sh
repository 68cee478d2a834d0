#!/bin/bash
# Round 2 session E: radix-sort A/B -- derived lines vs all-lines passes,
# tile size (keys per thread 16 / 24 / 32); GC time of the last of 4 frames.
set -u
for lib in paper_2401_09721_b200/_lib/libfgbd_b200.so tools/_lib_ipt24.so tools/_lib_ipt32.so; do
  for der in 1 0; do
    for a in "--kind ramp" "--kind ramp --order shuffle" "--kind constant"; do
      echo "== lib=$lib derived=$der $a"
      FGBD_LIB_PATH=$lib FGBD_SORT_DERIVED=$der timeout 120 python tools/profile_frame.py $a --frames 4 2>&1 | tail -1
    done
  done
done
echo done
