#!/bin/bash
# Round 2 session BE: k_slg per-block phase timeline.
set -u
echo "== ramp"; FGBD_SLG_TLOG=1 timeout 120 python tools/profile_frame.py --kind ramp --frames 2 2>&1 | grep -E "slg phase|frame" | tail -14
echo "== ramp shuffled"; FGBD_SLG_TLOG=1 timeout 120 python tools/profile_frame.py --kind ramp --order shuffle --frames 2 2>&1 | grep -E "slg phase|frame" | tail -29
