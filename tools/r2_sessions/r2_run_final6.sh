#!/bin/bash
# Round 2 session F6: the measurement set on the final state of the round.
set -u
O=gpurun_out/r2f6; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; cat $O/smoke.log
python bench.py > $O/bench_frame.json 2> $O/bench_frame.err; echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo "reference rc=$?"
python bench.py --kind constant --no-cpu-baseline > $O/bench_constant.json 2> $O/bench_constant.err
python bench.py --kind two-tone --no-cpu-baseline > $O/bench_twotone.json 2> $O/bench_twotone.err
python bench.py --workload video > $O/bench_video.json 2> $O/bench_video.err
python bench.py --workload video --static-geometry > $O/bench_video_static.json 2> $O/bench_video_static.err
python bench.py --workload ply > $O/bench_ply.json 2> $O/bench_ply.err
for p in 1 2 4 8; do timeout 300 python bench.py --workload slab --slab-ranks $p --steps 5 > $O/bench_slab_p$p.json 2> $O/bench_slab_p$p.err; done
for s in 5 10 20 30; do python bench.py --sigma $s --no-cpu-baseline --no-e2e >> $O/sigma_sweep_ramp.jsonl 2>>$O/sweep.err; python bench.py --kind two-tone --sigma $s --no-cpu-baseline --no-e2e >> $O/sigma_sweep_twotone.jsonl 2>>$O/sweep.err; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_l.log 2>&1; echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_lf_run --launch-skip 2 --launch-count 1 -o $O/lf_run python tools/profile_frame.py --frames 3 > $O/ncu_lf.log 2>&1; echo "ncu lf rc=$?"

python bench.py --points 100000 --no-e2e > $O/bench_100k.json 2> $O/bench_100k.err; echo "100k rc=$?"
for n in 4000000 8000000; do timeout 300 python tools/profile_frame.py --n $n --frames 3 > $O/profile_$n.txt 2>&1; tail -1 $O/profile_$n.txt; done
for p in 1 8; do timeout 300 python tools/slab_frame.py --ranks $p --frames 3 > $O/slab_frame_p$p.txt 2>&1; tail -1 $O/slab_frame_p$p.txt; done
echo done
ncu --set full --clock-control none --import-source on -k regex:"k_slg|k_rows|k_noise2" --launch-skip 3 --launch-count 3 -o $O/side python tools/profile_frame.py --frames 3 > $O/ncu_side.log 2>&1; echo "ncu side rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_constant.csv python tools/profile_frame.py --kind constant --frames 3 > $O/ncu_l2.log 2>&1; echo "launches constant rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_twotone.csv python tools/profile_frame.py --kind two-tone --frames 3 > $O/ncu_l3.log 2>&1; echo "launches two-tone rc=$?"
