#!/bin/bash
# Round 2 session BL: where the bench step's time goes outside the stages.
set -u
O=gpurun_out/r2bl; mkdir -p $O
python bench.py --no-cpu-baseline --no-e2e > $O/bench_frame.json 2> $O/bench_frame.err; echo "bench rc=$?"
python bench.py --kind two-tone --no-cpu-baseline --no-e2e > $O/bench_twotone.json 2> $O/bench_twotone.err; echo "bench2 rc=$?"
