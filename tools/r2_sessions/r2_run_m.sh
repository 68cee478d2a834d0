#!/bin/bash
set -u
for g in 0 1; do for a in "--kind ramp" "--kind two-tone" "--kind constant" "--kind ramp --order shuffle"; do
  echo "== rows_grid=$g $a"; FGBD_ROWS_GRID=$g timeout 120 python tools/profile_frame.py $a --frames 4 2>&1 | tail -1
done; done
