#!/bin/bash
# Round 2 session BY: k_noise2 with software-pipelined meta / slot loads (A/B).
set -u
for rep in 1 2; do
for lib in paper_2401_09721_b200/_lib/libfgbd_b200.so tools/_lib_FGBD_NE_PF_1.so tools/_lib_FGBD_NE_PF_1_FGBD_NE_MINB_5.so tools/_lib_FGBD_NE_PF_1_FGBD_NE_MINB_4.so; do
  for k in ramp constant; do
    echo "== lib=$lib $k"; FGBD_LIB_PATH=$lib timeout 120 python tools/profile_frame.py --kind $k --frames 4 2>&1 | tail -1
  done
done
done
