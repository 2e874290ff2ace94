#!/bin/bash
# bash scripts/gpu_4.sh TAG : 4-GPU parity (sync + async), configs[4] sweep, scale-family bench
TAG=${1:-q01}; N=4
OUT=gpurun_out/$TAG; mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533"
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > $OUT/pytest_multi.log 2>&1; echo "rc=$?" >> $OUT/pytest_multi.log
for S in 0 2 5; do
  timeout 300 $TR bench.py --gpus $N --workload cfg5 --slow $S --window 4 --warmup 3 > $OUT/ours_cfg5_s$S.json 2> $OUT/ours_cfg5_s$S.err
  timeout 300 $TR bench.py --gpus $N --workload cfg5 --slow $S --impl nccl --steps 200 --warmup 5 > $OUT/nccl_cfg5_s$S.json 2> $OUT/nccl_cfg5_s$S.err
done
timeout 300 $TR bench.py --gpus $N --steps 100 --warmup 5 > $OUT/bench_default.json 2> $OUT/bench_default.err
timeout 300 $TR bench.py --gpus $N --impl reference --steps 3 --warmup 3 > $OUT/reference_default.json 2> $OUT/reference_default.err
echo done > $OUT/DONE
