#!/bin/bash
# bash scripts/gpu_4_final2.sh TAG : on a 4-GPU box, every multi-GPU parity test, then the default
# multi-GPU bench (Inter-Intra layout) and the other multi-GPU workloads at N = 2 and 4 (ours vs
# NCCL all-reduce), bf16 Inter-Intra, configs[4] (cfg5) at slow factors 0/2/5, reference arm.
TAG=${1:-f02}; N=4
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider > $OUT/pytest_multi.log 2>&1; echo "rc=$?" >> $OUT/pytest_multi.log
for NG in 2 4; do
  T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29534"
  timeout 300 $T2 bench.py --gpus $NG > $OUT/ours_default_n$NG.json 2> $OUT/ours_default_n$NG.err
  timeout 300 $T2 bench.py --gpus $NG --impl nccl --steps 100 --warmup 5 > $OUT/nccl_default_n$NG.json 2> $OUT/nccl_default_n$NG.err
  for WL in cfg2 cfg3 cfg4 cfg2iibf16; do
    timeout 300 $T2 bench.py --gpus $NG --steps 100 --warmup 5 --workload $WL --no-cpu-baseline > $OUT/ours_${WL}_n$NG.json 2> $OUT/ours_${WL}_n$NG.err
    if [ $WL != cfg2iibf16 ]; then
      timeout 300 $T2 bench.py --gpus $NG --steps 100 --warmup 5 --workload $WL --impl nccl > $OUT/nccl_${WL}_n$NG.json 2> $OUT/nccl_${WL}_n$NG.err
    fi
  done
done
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533"
for S in 0 2 5; do
  timeout 300 $TR bench.py --gpus $N --workload cfg5 --slow $S --window 4 --warmup 3 > $OUT/ours_cfg5_s$S.json 2> $OUT/ours_cfg5_s$S.err
  timeout 300 $TR bench.py --gpus $N --workload cfg5 --slow $S --impl nccl --steps 200 --warmup 5 > $OUT/nccl_cfg5_s$S.json 2> $OUT/nccl_cfg5_s$S.err
done
timeout 300 $TR bench.py --gpus $N --impl reference --steps 3 --warmup 3 > $OUT/reference_default_n4.json 2> $OUT/reference_default_n4.err
echo done > $OUT/DONE
