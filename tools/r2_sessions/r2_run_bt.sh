#!/bin/bash
# Round 2 session BT: no elapsed-time query after a device-output frame
# (t_d2h = 0: no download) -- bench repeats.
set -u
O=gpurun_out/r2bt; mkdir -p $O
timeout 600 python -m pytest tests/test_reuse.py tests/test_boundary.py -m gpu -q -p no:cacheprovider > $O/tests.log 2>&1; echo "tests rc=$?"; tail -1 $O/tests.log
for rep in 1 2 3; do
python bench.py --no-cpu-baseline --no-e2e > $O/bench_$rep.json 2> $O/bench_$rep.err
python -c "import json; d=json.loads(open('$O/bench_$rep.json').read().strip().splitlines()[-1]); print('rep $rep', round(d['value'],1), d['ms_per_step'], d['stage_ms']['in_library_ms'])"
done
