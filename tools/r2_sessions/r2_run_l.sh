#!/bin/bash
# Round 2 session L: ncu evidence for the round-2 kernels (k_lf_run at 1M /
# 8M with size-aware rows, the derived sort pass, k_noise2, k_rows), the
# N = 2 self-launch harness check, and Morton row order on random clouds.
set -u
O=gpurun_out/r2l; mkdir -p $O
for n in 1000000 8000000; do
  ncu --set full --clock-control none --import-source on -k regex:k_lf_run --launch-skip 1 --launch-count 1 \
    -o $O/lf_run_$n python tools/profile_frame.py --n $n --frames 2 > $O/ncu_lf_$n.log 2>&1; echo "ncu lf $n rc=$?"
done
ncu --set full --clock-control none --import-source on -k regex:"k_onesweep|k_noise2|k_rows|k_neighbors|k_prep|k_mask" --launch-skip 0 --launch-count 20 \
    -o $O/side python tools/profile_frame.py --frames 1 > $O/ncu_side.log 2>&1; echo "ncu side rc=$?"
FGBD_BENCH_SHARED_GPU=1 FGBD_DEVICE=0 timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > $O/harness_n2.json 2> $O/harness_n2.err; echo "harness n2 rc=$?"; tail -c 400 $O/harness_n2.json
for o in "--order asis" "--order morton"; do for r in 1 0; do echo "== constant reorder=$r $o"; FGBD_REORDER=$r timeout 120 python tools/profile_frame.py --kind constant $o --frames 4 2>&1 | tail -1; done; done
echo done
