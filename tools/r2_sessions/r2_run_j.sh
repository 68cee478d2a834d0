#!/bin/bash
set -u
O=gpurun_out/r2j; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "slab" > $O/slab_tests.log 2>&1; echo "slab tests rc=$?"; tail -2 $O/slab_tests.log
for p in 1 8; do timeout 300 python bench.py --workload slab --slab-ranks $p --steps 5 > $O/bench_slab_p$p.json 2> $O/bench_slab_p$p.err; echo "slab p$p rc=$?"; python -c "
import json;d=json.loads(open('$O/bench_slab_p$p.json').read().strip().splitlines()[-1]); print(d['value'], d['stage_ms'])"; done
