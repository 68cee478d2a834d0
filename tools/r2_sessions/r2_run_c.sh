#!/bin/bash
# Round 2 session C: full GPU suite, headline bench, slab bench (emulated
# P = 1/2/4/8, per-rank stage times), video with/without static geometry.
set -u
O=gpurun_out/r2c; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/gpu_tests.log
python bench.py > $O/bench_frame.json 2> $O/bench_frame.err; echo "bench rc=$?"
for p in 1 2 4 8; do timeout 300 python bench.py --workload slab --slab-ranks $p --steps 5 > $O/bench_slab_p$p.json 2> $O/bench_slab_p$p.err; echo "slab p$p rc=$?"; done
python bench.py --workload video > $O/bench_video.json 2> $O/bench_video.err; echo "video rc=$?"
python bench.py --workload video --static-geometry > $O/bench_video_static.json 2> $O/bench_video_static.err; echo "video static rc=$?"
echo done
