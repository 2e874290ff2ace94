#!/bin/bash
# bash scripts/gpu_k1.sh TAG : single-worker (singleton group, SGD only) launch, variant 5 vs 7, N=1
TAG=${1:-s1}; OUT=gpurun_out/$TAG; mkdir -p $OUT
for V in 5 7 5 7; do
  RP_PREDUCE_TMA=$V timeout 120 python bench.py --workload cfg3 --steps 200 --warmup 5 --no-cpu-baseline --e2e-steps 1 > $OUT/t.json 2> $OUT/t.err
  echo "V=$V $(python -c "
import json
d=json.loads([l for l in open('$OUT/t.json') if l.startswith('{')][0]); r=d['roofline']
print(d['ms_per_step'], r['kernel_ms_per_launch'], r['achieved'], r['algorithmic_bytes_per_launch'])")" >> $OUT/sweep.txt
done
for WL in cfg2 cfg2ii; do for V in 7 5; do
  RP_PREDUCE_TMA=$V timeout 120 python bench.py --workload $WL --steps 200 --warmup 5 --no-cpu-baseline --e2e-steps 1 > $OUT/t.json 2> $OUT/t.err
  echo "$WL V=$V $(python scripts/show_bench.py $OUT/t.json)" >> $OUT/sweep.txt
done; done
echo done > $OUT/DONE
