#!/bin/bash
# bash scripts/xgpu_sweep.sh TAG N "workloads" "ENV1;ENV2;..." : cross-kernel knob sweep (bench lines
# summarised by scripts/show_bench.py) into gpurun_out/TAG/sweep.txt
TAG=$1; N=$2; WLS=$3; VARIANTS=$4
OUT=gpurun_out/$TAG; mkdir -p $OUT
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29545"
IFS=';' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do
  for wl in $WLS; do
    env $v timeout 300 $T bench.py --gpus $N --workload $wl --steps 60 --e2e-steps 1 --no-extras 2>$OUT/err.txt | grep '^{' > $OUT/tmp.json
    echo "$wl [$v] $(python scripts/show_bench.py $OUT/tmp.json)" >> $OUT/sweep.txt
  done
done
