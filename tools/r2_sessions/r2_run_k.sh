#!/bin/bash
set -u
O=gpurun_out/r2k; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/gpu_tests.log
python bench.py --no-cpu-baseline > $O/bench_frame.json 2> $O/bench_frame.err; echo "bench rc=$?"
for t in 0 2 4 8; do FGBD_HOST_THREADS=$t python bench.py --no-cpu-baseline --steps 10 > $O/bench_ht$t.json 2>/dev/null; python -c "
import json;d=json.loads(open('$O/bench_ht$t.json').read().strip().splitlines()[-1]); print('threads=$t', round(d['value'],1), round(d['e2e']['value'],1), round(d['e2e_pageable']['value'],1))"; done
