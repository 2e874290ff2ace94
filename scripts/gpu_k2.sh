#!/bin/bash
# bash scripts/gpu_k2.sh TAG : variant tests (incl. forced variant 7), 1-GPU parity, and the
# 1-GPU benches after the size-based kernel choice
TAG=${1:-s2}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py tests/test_gpu_kernels.py -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for WL in cfg2 cfg2ii cfg2bf16 cfg3 cfg1; do
  timeout 120 python bench.py --workload $WL --steps 200 --warmup 5 --no-cpu-baseline --e2e-steps 1 > $OUT/t.json 2> $OUT/t.err
  echo "$WL $(python scripts/show_bench.py $OUT/t.json)" >> $OUT/sweep.txt
done
echo done > $OUT/DONE
