#!/bin/bash
# Round 2 session BC: phase timeline of k_slg (block 0, %globaltimer).
set -u
for k in ramp constant; do
  echo "== $k"; FGBD_SLG_TLOG=1 timeout 120 python tools/profile_frame.py --kind $k --frames 3 2>&1 | grep -E "slg tlog|frame" | tail -4
done
echo "== ramp shuffled"; FGBD_SLG_TLOG=1 timeout 120 python tools/profile_frame.py --kind ramp --order shuffle --frames 3 2>&1 | grep -E "slg tlog|frame" | tail -2
