#!/bin/bash
# bash scripts/gpu_bf16.sh TAG : 1-GPU parity (fp32 + bf16) and the bf16 / fp32 configs[1] benches
TAG=${1:-bf1}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_engine.py -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for WL in cfg2bf16 cfg2; do
  timeout 300 python bench.py --steps 200 --warmup 5 --workload $WL --cpu-budget 5 > $OUT/$WL.json 2> $OUT/$WL.err
  echo "$WL $(python scripts/show_bench.py $OUT/$WL.json)" >> $OUT/sweep.txt
done
CMD="python bench.py --steps 8 --warmup 3 --no-cpu-baseline --e2e-steps 1 --workload cfg2bf16"
if timeout 300 $CMD > $OUT/ncu_plain.log 2>&1; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:preduce_ -s 6 -c 1 -o $OUT/prof $CMD > $OUT/ncu_full.log 2>&1
fi
echo done > $OUT/DONE
