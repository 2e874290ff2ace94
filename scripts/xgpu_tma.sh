#!/bin/bash
TAG=${1:-t01}; N=${2:-2}
OUT=gpurun_out/$TAG; mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533"
RP_XGPU_TMA=1 timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -p no:cacheprovider -k "not async and not momentum" > $OUT/pytest_tma.log 2>&1; echo "rc=$?" >> $OUT/pytest_tma.log
for REP in 1 2; do
for TMA in 0 1; do
 for WL in cfg3 cfg4 cfg2ii; do
   RP_XGPU_TMA=$TMA timeout 200 $TR bench.py --gpus $N --steps 50 --warmup 5 --workload $WL --e2e-steps 1 2>/dev/null | grep '^{' > $OUT/tmp.json
   echo "$WL TMA=$TMA $(python scripts/show_bench.py $OUT/tmp.json)" >> $OUT/sweep.txt
 done
done
done
RP_XGPU_TMA=1 RP_XGPU_PROFILE=$OUT/tl_cfg4 timeout 200 $TR bench.py --gpus $N --steps 20 --warmup 3 --workload cfg4 --e2e-steps 1 > /dev/null 2>&1
echo done >> $OUT/sweep.txt
