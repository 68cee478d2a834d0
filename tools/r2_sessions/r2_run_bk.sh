#!/bin/bash
# Round 2 session BK: one host wait at the end of a frame (control block D2H
# behind the last kernel): concurrency / reuse / parity tests and the bench.
set -u
O=gpurun_out/r2bk; mkdir -p $O
timeout 900 python -m pytest tests/test_concurrency_gpu.py tests/test_reuse.py tests/test_sequence.py tests/test_gpu_parity.py tests/test_device_finish.py -m gpu -x -q -p no:cacheprovider > $O/tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/tests.log
python bench.py --no-cpu-baseline > $O/bench_frame.json 2> $O/bench_frame.err; echo "bench rc=$?"
python bench.py --kind two-tone --no-cpu-baseline > $O/bench_twotone.json 2> $O/bench_twotone.err; echo "bench2 rc=$?"
