#!/bin/bash
# bash scripts/gpu_multi.sh TAG N "workload ..." [extra bench args]: N-GPU bench lines (ours + NCCL AR)
# for each workload, into gpurun_out/TAG/. Used from gpurun (--gpus N).
TAG=$1; N=$2; WLS=$3; shift 3
OUT=gpurun_out/$TAG; mkdir -p $OUT
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29541"
for wl in $WLS; do
  timeout 300 $T bench.py --gpus $N --workload $wl "$@" > $OUT/ours_${wl}_n$N.json 2> $OUT/ours_${wl}_n$N.err
  timeout 300 $T bench.py --gpus $N --workload $wl --impl nccl "$@" > $OUT/ar_${wl}_n$N.json 2> $OUT/ar_${wl}_n$N.err
done
echo done > $OUT/DONE
