#!/bin/bash
# A/B on one box: tools/ab.sh "<label>=<env assignments>" ... ; each runs 3 alternating rounds.
# Example: tools/ab.sh "base=FGBD_LIB_PATH=profiles/lib_base.so" "new="
ARGS=${AB_ARGS:-"--frames 3"}
for r in 1 2 3; do
  for spec in "$@"; do
    label=${spec%%=*}; envs=${spec#*=}
    printf "%-10s " "$label"; env $envs python tools/profile_frame.py $ARGS | tail -1
  done
done
