#!/bin/bash
# Round 2 session BX: k_rows with software-pipelined candidate loads (A/B).
set -u
for rep in 1 2; do
for lib in paper_2401_09721_b200/_lib/libfgbd_b200.so tools/_lib_FGBD_ROWS_PF_1.so tools/_lib_FGBD_ROWS_PF_1_FGBD_ROWS_MINB_3.so; do
  for k in ramp constant; do
    echo "== lib=$lib $k"; FGBD_LIB_PATH=$lib timeout 120 python tools/profile_frame.py --kind $k --frames 4 2>&1 | tail -1
  done
  echo "== lib=$lib ramp shuffled"; FGBD_LIB_PATH=$lib timeout 120 python tools/profile_frame.py --kind ramp --order shuffle --frames 4 2>&1 | tail -1
done
done
