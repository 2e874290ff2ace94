#!/bin/bash
# bash scripts/gpu_xall.sh TAG : NVLink efficiency of the push kernel with one all-GPU group per step
TAG=${1:-xa1}
OUT=gpurun_out/$TAG; mkdir -p $OUT
for NG in 4 2 3; do
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 2953$NG"
  for WL in xall xall_vgg; do
    timeout 300 $TR bench.py --gpus $NG --steps 60 --warmup 5 --workload $WL --e2e-steps 1 > $OUT/${WL}_n$NG.json 2> $OUT/${WL}_n$NG.err
    echo "$WL n=$NG $(python scripts/show_bench.py $OUT/${WL}_n$NG.json)" >> $OUT/sweep.txt
    timeout 300 $TR bench.py --gpus $NG --steps 60 --warmup 5 --workload $WL --impl nccl > $OUT/nccl_${WL}_n$NG.json 2> $OUT/nccl_${WL}_n$NG.err
    echo "$WL n=$NG $(python scripts/show_bench.py $OUT/nccl_${WL}_n$NG.json)" >> $OUT/sweep.txt
  done
  RP_XGPU_PROFILE=$OUT/tl_n$NG timeout 300 $TR bench.py --gpus $NG --steps 10 --warmup 3 --workload xall --e2e-steps 1 > /dev/null 2>&1
  python scripts/xgpu_timeline.py $OUT/tl_n$NG.* > $OUT/timeline_n$NG.txt 2>&1
done
NG=4; TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29539"
for CPS in 1 2 3; do
  for CH in 4096 8192 16384 32768; do
    RP_XGPU_CHUNK_F4=$CH RP_XGPU_CTAS_PER_SM=$CPS timeout 200 $TR bench.py --gpus 4 --steps 40 --warmup 3 --workload xall --e2e-steps 1 > $OUT/tmp.json 2>/dev/null
    echo "xall n=4 CPS=$CPS CH=$CH $(python scripts/show_bench.py $OUT/tmp.json)" >> $OUT/sweep.txt
  done
done
echo done > $OUT/DONE
