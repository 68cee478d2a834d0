#!/bin/bash
# Round 2 session B: partitioned slab parity (GPU), 8M slab parity, slab bench
# at emulated P = 1/2/4/8, and the 8M filter's row-assignment knob.
set -u
O=gpurun_out/r2b; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "slab" > $O/slab_tests.log 2>&1; echo "slab tests rc=$?"; tail -15 $O/slab_tests.log
timeout 900 python -m pytest tests/test_frame_8m.py -q -p no:cacheprovider -x > $O/t8m.log 2>&1; echo "8m tests rc=$?"; tail -5 $O/t8m.log
for p in 1 2 4 8; do timeout 300 python bench.py --workload slab --slab-ranks $p --steps 5 > $O/bench_slab_p$p.json 2> $O/bench_slab_p$p.err; echo "slab p$p rc=$?"; tail -c 600 $O/bench_slab_p$p.json; done
for ch in 1 0; do for n in 1000000 8000000; do echo "== chunk=$ch n=$n"; FGBD_LF_CHUNK=$ch timeout 300 python tools/profile_frame.py --n $n --frames 3 2>&1 | tail -1; done; done
echo done
