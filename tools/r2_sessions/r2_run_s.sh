#!/bin/bash
set -u
O=gpurun_out/r2s; mkdir -p $O
timeout 600 python -m pytest tests/test_device_finish.py -q -p no:cacheprovider -x > $O/finish_tests.log 2>&1; echo "finish tests rc=$?"; tail -3 $O/finish_tests.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/gpu_tests.log
for a in "--kind ramp" "--kind two-tone" "--kind constant"; do echo "== $a"; timeout 120 python tools/profile_frame.py $a --frames 4 2>&1 | tail -1; done
python bench.py --no-cpu-baseline > $O/bench_frame.json 2>/dev/null; python -c "import json; d=json.loads(open('$O/bench_frame.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['e2e_pageable']['value'])"
for w in 2 3 4; do python bench.py --workload video --workers $w > $O/bench_video_w$w.json 2>/dev/null; python -c "import json; print('video w=$w', json.loads(open('$O/bench_video_w$w.json').read().strip().splitlines()[-1])['value'])"; done
python bench.py --workload video --static-geometry > $O/bench_video_static.json 2>/dev/null; python -c "import json; print('video static', json.loads(open('$O/bench_video_static.json').read().strip().splitlines()[-1])['value'])"
