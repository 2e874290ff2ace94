#!/bin/bash
# bash scripts/gpu_cfg5b.sh TAG N : configs[4] ours vs NCCL AR at slow factors 0/2/5 (host-sleep compute)
TAG=${1:-h02}; N=${2:-4}
OUT=gpurun_out/$TAG; mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533"
for S in 0 2 5; do
  timeout 300 $TR bench.py --gpus $N --workload cfg5 --slow $S --window 4 --warmup 3 > $OUT/ours_cfg5_s$S.json 2> $OUT/ours_cfg5_s$S.err
  timeout 300 $TR bench.py --gpus $N --workload cfg5 --slow $S --impl nccl --steps 200 --warmup 5 > $OUT/nccl_cfg5_s$S.json 2> $OUT/nccl_cfg5_s$S.err
done
echo done > $OUT/DONE
