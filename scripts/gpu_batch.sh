#!/bin/bash
# bash scripts/gpu_batch.sh TAG : tile ids per atomic (RP_DYN_BATCH) of the dynamic-tile kernel, N=1
TAG=${1:-b1}; OUT=gpurun_out/$TAG; mkdir -p $OUT
for REP in 1 2; do
for B in 0 1 2 4 8; do
  for WL in cfg2 cfg2ii cfg2bf16; do
    RP_DYN_BATCH=$B timeout 120 python bench.py --workload $WL --steps 200 --warmup 5 --no-cpu-baseline --e2e-steps 1 > $OUT/t.json 2> $OUT/t.err
    echo "B=$B $WL $(python scripts/show_bench.py $OUT/t.json)" >> $OUT/sweep.txt
  done
done
done
echo done > $OUT/DONE
