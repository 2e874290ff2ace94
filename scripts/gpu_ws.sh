#!/bin/bash
# bash scripts/gpu_ws.sh TAG : parity + sweep of the warp-specialized intra-GPU kernel (variants 5, 6)
TAG=${1:-ws1}
OUT=gpurun_out/$TAG; mkdir -p $OUT
for V in 5 6; do
  RP_PREDUCE_TMA=$V RP_PREDUCE_BF16=$V timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py -q -x -p no:cacheprovider > $OUT/pytest_$V.log 2>&1; echo rc=$? >> $OUT/pytest_$V.log
done
for REP in 1 2; do
  for V in 3 5 6; do
    for WL in cfg2 cfg2bf16 cfg2ii; do
      RP_PREDUCE_TMA=$V RP_PREDUCE_BF16=$V timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --e2e-steps 1 --workload $WL > $OUT/t.json 2>/dev/null
      echo "$WL V=$V $(python scripts/show_bench.py $OUT/t.json)" >> $OUT/sweep.txt
    done
  done
done
echo done > $OUT/DONE
