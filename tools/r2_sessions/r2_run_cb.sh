#!/bin/bash
# Round 2 session CB: a free device takes the frame without waiting for the
# coordinates to land -- concurrency / reuse / sequence tests, e2e, video.
set -u
O=gpurun_out/r2cb; mkdir -p $O
timeout 900 python -m pytest tests/test_concurrency_gpu.py tests/test_reuse.py tests/test_sequence.py tests/test_gpu_parity.py tests/test_ply.py -m gpu -x -q -p no:cacheprovider > $O/tests.log 2>&1; echo "tests rc=$?"; tail -1 $O/tests.log
timeout 300 python tools/concurrency_repro.py | tail -2
for rep in 1 2; do
python bench.py --no-cpu-baseline --steps 5 > $O/bench_$rep.json 2> $O/bench_$rep.err
python -c "import json; d=json.loads(open('$O/bench_$rep.json').read().strip().splitlines()[-1]); print('rep $rep', round(d['value'],1), d['e2e']['value'], d['e2e_pageable']['value'])"
python bench.py --workload video > $O/video_$rep.json 2> $O/video_$rep.err; python -c "import json; d=json.loads(open('$O/video_$rep.json').read().strip().splitlines()[-1]); print('video', round(d['value'],1))"
python bench.py --workload video --static-geometry > $O/videos_$rep.json 2> $O/videos_$rep.err; python -c "import json; d=json.loads(open('$O/videos_$rep.json').read().strip().splitlines()[-1]); print('video static', round(d['value'],1))"
python bench.py --workload ply > $O/ply_$rep.json 2> $O/ply_$rep.err; python -c "import json; d=json.loads(open('$O/ply_$rep.json').read().strip().splitlines()[-1]); print('ply', round(d['value'],1))"
done
