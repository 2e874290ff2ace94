#!/bin/bash
TAG=${1:-s04}; N=${2:-2}
OUT=gpurun_out/$TAG; mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533"
for ORD in 0 1; do
 for WL in cfg3 cfg4; do
  for CH in 8192 16384; do
   RP_XGPU_ORDER=$ORD RP_XGPU_CHUNK_F4=$CH timeout 200 $TR bench.py --gpus $N --steps 30 --warmup 3 --workload $WL --e2e-steps 1 2>/dev/null | grep '^{' > $OUT/tmp.json
   echo "$WL ORD=$ORD CH=$CH $(python scripts/show_bench.py $OUT/tmp.json)" >> $OUT/sweep.txt
  done
 done
done
RP_XGPU_ORDER=1 RP_XGPU_PROFILE=$OUT/tl_cfg3 timeout 200 $TR bench.py --gpus $N --steps 20 --warmup 3 --workload cfg3 --e2e-steps 1 > /dev/null 2>&1
RP_XGPU_ORDER=1 timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -p no:cacheprovider -k "not async" > $OUT/pytest_multi.log 2>&1; echo "rc=$?" >> $OUT/pytest_multi.log
echo done >> $OUT/sweep.txt
