#!/bin/bash
# Round 2 session BP: decide-before-sweep when a stop is one step away
# (FGBD_LF_HOLD) A/B; the frame-tail fix for multi-context video; the
# scan-line front-end boundary tests; full GPU suite.
set -u
O=gpurun_out/r2bp; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/tests.log
for rep in 1 2; do
for lib in paper_2401_09721_b200/_lib/libfgbd_b200.so tools/_lib_nohold.so; do
  for k in ramp two-tone constant; do
    echo "== lib=$lib $k"; FGBD_LIB_PATH=$lib timeout 120 python tools/profile_frame.py --kind $k --frames 4 2>&1 | tail -1
  done
done
done
python bench.py --workload video > $O/bench_video.json 2> $O/bench_video.err; echo "video rc=$?"
python bench.py --workload video --static-geometry > $O/bench_video_static.json 2> $O/bench_video_static.err; echo "video static rc=$?"
python bench.py --no-cpu-baseline > $O/bench_frame.json 2> $O/bench_frame.err; echo "bench rc=$?"
python bench.py --kind two-tone --no-cpu-baseline > $O/bench_twotone.json 2> $O/bench_twotone.err; echo "bench2 rc=$?"
python bench.py --kind constant --no-cpu-baseline > $O/bench_constant.json 2> $O/bench_constant.err; echo "bench3 rc=$?"
