#!/bin/bash
set -u
O=gpurun_out/r2aa; mkdir -p $O
export FGBD_BENCH_SHARED_GPU=1 FGBD_DEVICE=0
timeout 600 python bench.py --gpus 2 --steps 4 --warmup 3 > $O/frame_n2.json 2> $O/frame_n2.err; echo "frame n2 rc=$?"; tail -c 300 $O/frame_n2.json
timeout 600 python bench.py --gpus 2 --steps 4 --warmup 3 --workload video --frames 60 > $O/video_n2.json 2> $O/video_n2.err; echo "video n2 rc=$?"; tail -c 300 $O/video_n2.json
timeout 600 python bench.py --gpus 2 --impl reference --steps 1 --warmup 1 --n 100000 > $O/ref_n2.json 2> $O/ref_n2.err; echo "ref n2 rc=$?"; tail -c 300 $O/ref_n2.json
