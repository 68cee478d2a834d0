#!/bin/bash
set -u
O=gpurun_out/r2y; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/gpu_tests.log
for a in "--kind ramp" "--kind constant" "--kind two-tone" "--kind ramp --order shuffle" "--kind ramp --n 8000000" "--kind constant --n 4000000"; do echo "== $a"; timeout 120 python tools/profile_frame.py $a --frames 4 2>&1 | tail -1; done
python bench.py --kind constant --no-cpu-baseline > $O/bench_constant.json 2>/dev/null; python -c "import json; d=json.loads(open('$O/bench_constant.json').read().strip().splitlines()[-1]); print('constant', d['value'], d['e2e']['value'], d['roofline']['frac'])"
