#!/bin/bash
# bash scripts/gpu_cfg5.sh TAG N : async multi-GPU parity tests, then configs[4] (ours vs NCCL AR)
TAG=${1:-h01}; N=${2:-2}
OUT=gpurun_out/$TAG; mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533"
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -p no:cacheprovider -k async > $OUT/pytest_async.log 2>&1; echo "rc=$?" >> $OUT/pytest_async.log
grep -q "rc=0" $OUT/pytest_async.log || exit 1
for S in 0 2 5; do
  timeout 300 $TR bench.py --gpus $N --workload cfg5 --slow $S --window 4 --warmup 3 > $OUT/ours_s$S.json 2> $OUT/ours_s$S.err
  timeout 300 $TR bench.py --gpus $N --workload cfg5 --slow $S --impl nccl --steps 200 --warmup 5 > $OUT/nccl_s$S.json 2> $OUT/nccl_s$S.err
done
echo done > $OUT/DONE
