#!/bin/bash
set -u
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "slab" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_frame_8m.py -q -p no:cacheprovider -x 2>&1 | tail -2
for p in 1 2 4 8; do echo "== 8M P=$p"; python tools/slab_frame.py --ranks $p --frames 3 | tail -1; done
echo "== 1M P=1"; python tools/slab_frame.py --n 1000000 --ranks 1 --frames 3 | tail -1
echo "== 1M P=8"; python tools/slab_frame.py --n 1000000 --ranks 8 --frames 3 | tail -1
