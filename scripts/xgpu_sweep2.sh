#!/bin/bash
# bash scripts/xgpu_sweep2.sh TAG N : parity tests, then knob sweep of the cross kernel
TAG=${1:-s02}; N=${2:-2}
OUT=gpurun_out/$TAG; mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533"
timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q -p no:cacheprovider > $OUT/pytest_multi.log 2>&1; echo "rc=$?" >> $OUT/pytest_multi.log
grep -q "rc=0" $OUT/pytest_multi.log || exit 1
for WL in cfg3 cfg4; do
 for CPS in 2; do
  for CH in 2048 4096 8192 16384 32768; do
    RP_XGPU_CHUNK_F4=$CH RP_XGPU_CTAS_PER_SM=$CPS timeout 200 $TR bench.py --gpus $N --steps 30 --warmup 3 --workload $WL --e2e-steps 1 2>/dev/null | grep '^{' > $OUT/tmp.json
    echo "$WL CPS=$CPS CH=$CH $(python scripts/show_bench.py $OUT/tmp.json)" >> $OUT/sweep.txt
  done
 done
done
RP_XGPU_PROFILE=$OUT/tl_cfg3 timeout 200 $TR bench.py --gpus $N --steps 20 --warmup 3 --workload cfg3 --e2e-steps 1 > /dev/null 2>&1
RP_XGPU_PROFILE=$OUT/tl_cfg4 timeout 200 $TR bench.py --gpus $N --steps 20 --warmup 3 --workload cfg4 --e2e-steps 1 > /dev/null 2>&1
echo done >> $OUT/sweep.txt
