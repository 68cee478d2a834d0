#!/bin/bash
# Round 2 session BZ: lines 2 / 3 through inverse orders (FGBD_SLG_INV):
# full GPU suite, A/B at 1M and 8M.
set -u
O=gpurun_out/r2bz; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
for rep in 1 2; do
for m in 1 0; do
  for k in ramp constant; do
    echo "== inv=$m $k"; FGBD_SLG_INV=$m timeout 120 python tools/profile_frame.py --kind $k --frames 4 2>&1 | tail -1
  done
  echo "== inv=$m ramp shuffled"; FGBD_SLG_INV=$m timeout 120 python tools/profile_frame.py --kind ramp --order shuffle --frames 4 2>&1 | tail -1
  echo "== inv=$m 8M"; FGBD_SLG_INV=$m timeout 200 python tools/profile_frame.py --n 8000000 --frames 3 2>&1 | tail -1
done
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_8m.csv python tools/profile_frame.py --n 8000000 --frames 2 > $O/ncu_l.log 2>&1; echo "launches rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_1m.csv python tools/profile_frame.py --frames 3 > $O/ncu_l1.log 2>&1; echo "launches rc=$?"
