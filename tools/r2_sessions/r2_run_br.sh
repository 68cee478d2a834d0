#!/bin/bash
# Round 2 session BR: host threads for pageable staging (e2e_pageable).
set -u
O=gpurun_out/r2br; mkdir -p $O
nproc; lscpu | grep -E "Model name|Socket|Core|Thread|NUMA node\(s\)" 
for t in 6 12 24; do
  FGBD_HOST_THREADS=$t python bench.py --no-cpu-baseline --steps 5 > $O/bench_t$t.json 2> $O/bench_t$t.err
  python -c "import json; d=json.loads(open('$O/bench_t$t.json').read().strip().splitlines()[-1]); print('threads $t', d['e2e']['value'], d['e2e_pageable']['value'])"
done
