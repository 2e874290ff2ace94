#!/bin/bash
# bash scripts/gpu_cfg2n2.sh TAG : cfg2 (plain GD over 8N workers) at N=2 under kernel-variant / split settings
TAG=${1:-c2}; OUT=gpurun_out/$TAG; mkdir -p $OUT
T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534"
for REP in 1 2; do
for E in "RP_PREDUCE_TMA=5" "RP_PREDUCE_TMA=7" "RP_XGPU_SPLIT=0" "RP_PREDUCE_TMA=5 RP_XGPU_SPLIT=0"; do
  env $E timeout 200 $T2 bench.py --gpus 2 --workload cfg2 --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 1 > $OUT/t.json 2> $OUT/t.err
  echo "$E $(python scripts/show_bench.py $OUT/t.json)" >> $OUT/sweep.txt
done
done
echo done > $OUT/DONE
