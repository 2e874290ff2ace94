#!/bin/bash
# Multi-GPU call: parity tests, benches with the cross-kernel timeline, NCCL baseline.
# Usage: bash scripts/gpu_multi2.sh TAG N [workloads...]
TAG=${1:-m01}; N=${2:-2}; shift 2
WLS=${@:-cfg3 cfg4 cfg2}
OUT=gpurun_out/$TAG; mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533"
timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q -p no:cacheprovider > $OUT/pytest_multi.log 2>&1; echo "rc=$?" >> $OUT/pytest_multi.log
for WL in $WLS; do
  RP_XGPU_PROFILE=$OUT/tl_$WL timeout 300 $TR bench.py --gpus $N --steps 50 --warmup 5 --workload $WL > $OUT/bench_${WL}.json 2> $OUT/bench_${WL}.err; echo "rc=$?" >> $OUT/bench_${WL}.err
  timeout 300 $TR bench.py --gpus $N --steps 50 --warmup 5 --workload $WL --impl nccl > $OUT/nccl_${WL}.json 2> $OUT/nccl_${WL}.err; echo "rc=$?" >> $OUT/nccl_${WL}.err
done
echo done > $OUT/DONE
