#!/bin/bash
# Round 2 session BS: pageable colours staged right behind the coordinates
# with their DMA pipelined (side stream) -- e2e_pageable; reuse / parity tests.
set -u
O=gpurun_out/r2bs; mkdir -p $O
timeout 900 python -m pytest tests/test_reuse.py tests/test_gpu_parity.py tests/test_sequence.py tests/test_concurrency_gpu.py tests/test_ply.py -m gpu -x -q -p no:cacheprovider > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
for rep in 1 2; do
python bench.py --no-cpu-baseline --steps 5 > $O/bench_$rep.json 2> $O/bench_$rep.err
python -c "import json; d=json.loads(open('$O/bench_$rep.json').read().strip().splitlines()[-1]); print('rep $rep', round(d['value'],1), d['e2e']['value'], d['e2e_pageable']['value'])"
done
python bench.py --workload ply > $O/bench_ply.json 2> $O/bench_ply.err; echo "ply rc=$?"; python -c "import json; d=json.loads(open('$O/bench_ply.json').read().strip().splitlines()[-1]); print('ply', d['value'])"
