#!/bin/bash
set -u
O=gpurun_out/r2n; mkdir -p $O
python tools/slab_frame.py --ranks 1 --frames 2
for p in 1 8; do
ncu --set full --clock-control none --import-source on -k regex:k_lf_slab --launch-skip 1 --launch-count 1 \
    -o $O/lf_slab_p$p python tools/slab_frame.py --ranks $p --frames 2 > $O/ncu_slab_p$p.log 2>&1; echo "ncu slab p$p rc=$?"
done
