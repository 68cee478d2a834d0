#!/bin/bash
# Round 2 session D: derived-line sort -- graph / sort parity first, then the
# full suite, then GC timings (ramp raster order, shuffled, constant).
set -u
O=gpurun_out/r2d; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "radix or graph or perm or scan or order" > $O/sort_tests.log 2>&1; echo "sort tests rc=$?"; tail -5 $O/sort_tests.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -5 $O/gpu_tests.log
for a in "--kind ramp" "--kind ramp --order shuffle" "--kind constant" "--kind two-tone"; do echo "== $a"; timeout 300 python tools/profile_frame.py $a --frames 4 2>&1 | tail -1; done
python bench.py --no-cpu-baseline > $O/bench_frame.json 2> $O/bench_frame.err; echo "bench rc=$?"; tail -c 300 $O/bench_frame.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python tools/profile_frame.py --frames 3 > $O/ncu_l.log 2>&1; echo "launches rc=$?"
echo done
