#!/bin/bash
# Round 2 session BD: k_slg with the relaxed-spin grid barrier (timeline),
# and k_lf_run's barrier A/B (grid_barrier vs cooperative_groups grid.sync).
set -u
for k in ramp constant; do
  echo "== tlog $k"; FGBD_SLG_TLOG=1 timeout 120 python tools/profile_frame.py --kind $k --frames 3 2>&1 | grep -E "slg tlog|frame" | tail -2
done
for rep in 1 2 3; do
for lib in paper_2401_09721_b200/_lib/libfgbd_b200.so tools/_lib_bar0.so; do
  for k in ramp two-tone constant; do
    echo "== lib=$lib $k"; FGBD_LIB_PATH=$lib timeout 120 python tools/profile_frame.py --kind $k --frames 4 2>&1 | tail -1
  done
done
done
for lib in paper_2401_09721_b200/_lib/libfgbd_b200.so tools/_lib_bar0.so; do
  echo "== lib=$lib 8M"; FGBD_LIB_PATH=$lib timeout 200 python tools/profile_frame.py --n 8000000 --frames 3 2>&1 | tail -1
done
