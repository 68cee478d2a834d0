# N>1 harness check on a one-GPU box (bench.py FGBD_BENCH_SHARED_GPU): two
# ranks on GPU 0 over gloo, independent frames.  Exercises the torchrun path
# the driver's scaling run takes; the numbers are not bench values.
set -u
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
export FGBD_BENCH_SHARED_GPU=1 FGBD_DEVICE=0  # worker threads default to FGBD_DEVICE
$TR --master-port 29511 bench.py --gpus 2 --steps 4 --warmup 3; echo "frame rc=$?"
$TR --master-port 29512 bench.py --gpus 2 --steps 4 --warmup 3 --workload video --frames 60; echo "video rc=$?"
$TR --master-port 29513 bench.py --impl reference --gpus 2 --steps 1 --warmup 1; echo "reference rc=$?"
