#!/bin/bash
# Round 2, first GPU session: full GPU suite, N=1 bench lines (ramp default,
# constant kind), ncu of k_lf_run at 1M/4M/8M.
set -u
O=gpurun_out/r2a; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/gpu_tests.log
python bench.py > $O/bench_frame.json 2> $O/bench_frame.err; echo "bench rc=$?"
python bench.py --kind constant --no-cpu-baseline > $O/bench_constant.json 2> $O/bench_constant.err; echo "bench constant rc=$?"
python bench.py --workload slab > $O/bench_slab.json 2> $O/bench_slab.err; echo "slab rc=$?"
for n in 1000000 4000000 8000000; do
  ncu --set full --clock-control none --import-source on -k regex:k_lf_run --launch-skip 1 --launch-count 1 \
    -o $O/lf_run_$n python tools/profile_frame.py --n $n --frames 2 > $O/ncu_lf_$n.log 2>&1; echo "ncu $n rc=$?"
done
ncu --set full --clock-control none --import-source on -k regex:k_lf_run --launch-skip 1 --launch-count 1 \
    -o $O/lf_run_constant python tools/profile_frame.py --kind constant --frames 2 > $O/ncu_lf_constant.log 2>&1; echo "ncu constant rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_l.log 2>&1; echo "launches rc=$?"
echo done
