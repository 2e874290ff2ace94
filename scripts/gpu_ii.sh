#!/bin/bash
# bash scripts/gpu_ii.sh TAG : cfg2ii (Inter-Intra) at N=2: split cap x aux-stream priority, and the
# cross kernel's item timeline of the last inter step (RP_XGPU_PROFILE)
TAG=${1:-ii1}; OUT=gpurun_out/$TAG; mkdir -p $OUT
T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534"
for SP in 296 148; do
for PR in 0 1 -1; do
  RP_XGPU_SPLIT=$SP RP_AUX_PRIO=$PR timeout 200 $T2 bench.py --gpus 2 --workload cfg2ii --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 1 > $OUT/t.json 2> $OUT/t.err
  echo "split=$SP prio=$PR $(python scripts/show_bench.py $OUT/t.json)" >> $OUT/sweep.txt
done
done
RP_XGPU_PROFILE=$OUT/tl timeout 200 $T2 bench.py --gpus 2 --workload cfg2ii --steps 11 --warmup 5 --no-cpu-baseline --e2e-steps 1 > $OUT/tl.json 2> $OUT/tl.err
python scripts/xgpu_timeline.py $OUT/tl.0 $OUT/tl.1 > $OUT/timeline.txt 2>&1
echo done > $OUT/DONE
