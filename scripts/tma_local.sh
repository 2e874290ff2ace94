#!/bin/bash
# Sweep of the intra-GPU TMA kernel variants (RP_PREDUCE_TMA=v) against the LDG kernel (v=0).
OUT=gpurun_out/$1; mkdir -p $OUT
for V in ${PARITY_VARIANTS:-3 4 5}; do
  RP_PREDUCE_TMA=$V timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > $OUT/pytest_$V.log 2>&1; echo rc=$? >> $OUT/pytest_$V.log
done
for REP in 1 2; do
for T in ${VARIANTS:-0 1 2 3 4 5}; do
  for WL in cfg2 cfg2ii; do
    RP_PREDUCE_TMA=$T python bench.py --steps 200 --warmup 5 --no-cpu-baseline --e2e-steps 1 --workload $WL 2>/dev/null | grep '^{' > $OUT/t.json
    echo "$WL TMA=$T $(python scripts/show_bench.py $OUT/t.json)" >> $OUT/sweep.txt
  done
done
done
