#!/bin/bash
set -u
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "slab" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_frame_8m.py -q -p no:cacheprovider -x 2>&1 | tail -2
for p in 1 8; do echo "== 8M P=$p"; python tools/slab_frame.py --ranks $p --frames 3 | tail -1; done
