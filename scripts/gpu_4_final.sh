#!/bin/bash
# bash scripts/gpu_4_final.sh TAG : full GPU suite on 4 GPUs, then every multi-GPU workload at
# N = 2 and 4 (ours vs NCCL all-reduce), and configs[4] (cfg5) at slow factors 0/2/5.
TAG=${1:-f01}; N=4
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
for NG in 2 4; do
  T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29534"
  for WL in cfg2 cfg2ii cfg3 cfg4; do
    timeout 300 $T2 bench.py --gpus $NG --steps 100 --warmup 5 --workload $WL > $OUT/ours_${WL}_n$NG.json 2> $OUT/ours_${WL}_n$NG.err
    if [ $WL != cfg2ii ]; then
      timeout 300 $T2 bench.py --gpus $NG --steps 100 --warmup 5 --workload $WL --impl nccl > $OUT/nccl_${WL}_n$NG.json 2> $OUT/nccl_${WL}_n$NG.err
    fi
  done
done
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533"
for S in 0 2 5; do
  timeout 300 $TR bench.py --gpus $N --workload cfg5 --slow $S --window 4 --warmup 3 > $OUT/ours_cfg5_s$S.json 2> $OUT/ours_cfg5_s$S.err
  timeout 300 $TR bench.py --gpus $N --workload cfg5 --slow $S --impl nccl --steps 200 --warmup 5 > $OUT/nccl_cfg5_s$S.json 2> $OUT/nccl_cfg5_s$S.err
done
timeout 300 $TR bench.py --gpus $N --impl reference --steps 3 --warmup 3 > $OUT/reference_default.json 2> $OUT/reference_default.err
echo done > $OUT/DONE
