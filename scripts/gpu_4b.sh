#!/bin/bash
# bash scripts/gpu_4b.sh TAG : full GPU suite on 4 GPUs, Inter-Intra and random-GG benches
TAG=${1:-q03}; N=4
OUT=gpurun_out/$TAG; mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
for NG in 2 4; do
  T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29534"
  timeout 300 $T2 bench.py --gpus $NG --steps 100 --warmup 5 --workload cfg2ii > $OUT/cfg2ii_n$NG.json 2> $OUT/cfg2ii_n$NG.err
done
timeout 300 python bench.py --steps 100 --warmup 5 --workload cfg2ii --no-cpu-baseline > $OUT/cfg2ii_n1.json 2> $OUT/cfg2ii_n1.err
for S in 0 2 5; do
  timeout 300 $TR bench.py --gpus $N --workload cfg5 --slow $S --window 4 --warmup 3 --gg random --k 2 > $OUT/adpsgd_cfg5_s$S.json 2> $OUT/adpsgd_cfg5_s$S.err
  timeout 300 $TR bench.py --gpus $N --workload cfg5 --slow $S --window 4 --warmup 3 --gg random > $OUT/rgg_cfg5_s$S.json 2> $OUT/rgg_cfg5_s$S.err
done
echo done > $OUT/DONE
