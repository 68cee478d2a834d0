#!/bin/bash
set -u
O=gpurun_out/r2r; mkdir -p $O
timeout 600 python -m pytest tests/test_device_finish.py -q -p no:cacheprovider -x > $O/finish_tests.log 2>&1; echo "finish tests rc=$?"; tail -15 $O/finish_tests.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -4 $O/gpu_tests.log
for f in 1 0; do for a in "--kind ramp" "--kind two-tone" "--kind constant"; do
  echo "== fold=$f $a"; FGBD_MASK_FOLD=$f timeout 120 python tools/profile_frame.py $a --frames 4 2>&1 | tail -1
done; done
python bench.py --no-cpu-baseline > $O/bench_frame.json 2>/dev/null; tail -c 200 $O/bench_frame.json
python bench.py --workload video > $O/bench_video.json 2>/dev/null; python -c "import json; print(json.loads(open('$O/bench_video.json').read().strip().splitlines()[-1])['value'])"
