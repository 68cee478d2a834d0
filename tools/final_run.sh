set -x
mkdir -p gpurun_out/r1f
python bench.py > gpurun_out/r1f/bench_frame.json 2> gpurun_out/r1f/bench_frame.err
python bench.py --workload video > gpurun_out/r1f/bench_video.json 2> gpurun_out/r1f/bench_video.err
python bench.py --workload video --no-reuse > gpurun_out/r1f/bench_video_noreuse.json 2> gpurun_out/r1f/bench_video_noreuse.err
python bench.py --workload ply > gpurun_out/r1f/bench_ply.json 2> gpurun_out/r1f/bench_ply.err
python bench.py --workload slab > gpurun_out/r1f/bench_slab.json 2> gpurun_out/r1f/bench_slab.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r1f/bench_reference.json 2> gpurun_out/r1f/bench_reference.err
for k in ramp two-tone; do for s in 5 10 20 30; do python bench.py --kind $k --sigma $s --no-cpu-baseline >> gpurun_out/r1f/sigma_sweep_$k.jsonl 2>>gpurun_out/r1f/sweep.err; done; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1f/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r1f/ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_lf_run --launch-skip 2 --launch-count 1 -o gpurun_out/r1f/lf_run python tools/profile_frame.py --frames 3 > gpurun_out/r1f/ncu_lf.log 2>&1
echo done
