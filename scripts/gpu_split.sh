#!/bin/bash
# bash scripts/gpu_split.sh TAG : parity of the dynamic-tile intra-GPU kernel (variant 7) and of
# the split launch (cross kernel beside the intra-GPU kernel on a second stream), then sweeps:
# intra variant 5 vs 7 at N = 1, cross-kernel CTA budget RP_XGPU_SPLIT (0 = fused L items) at N = 2/4.
TAG=${1:-split1}
OUT=gpurun_out/$TAG; mkdir -p $OUT
NG=$(nvidia-smi -L | wc -l)
RP_PREDUCE_TMA=7 RP_PREDUCE_BF16=7 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_engine.py -q -x -p no:cacheprovider > $OUT/pytest_v7.log 2>&1; echo "rc=$?" >> $OUT/pytest_v7.log
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -x -p no:cacheprovider -k "not nvls" > $OUT/pytest_multi.log 2>&1; echo "rc=$?" >> $OUT/pytest_multi.log
for V in 5 6 7; do
  for WL in cfg2 cfg2ii cfg2bf16; do
    RP_PREDUCE_TMA=$V RP_PREDUCE_BF16=$V timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --e2e-steps 1 --workload $WL > $OUT/t.json 2>/dev/null
    echo "n1 $WL V=$V $(python scripts/show_bench.py $OUT/t.json)" >> $OUT/sweep.txt
  done
done
for N in 2 4; do
  [ $N -gt $NG ] && continue
  T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29534"
  for SP in ${SPLITS:-0 74 148 296}; do
    for WL in cfg2ii cfg2; do
      RP_XGPU_SPLIT=$SP timeout 200 $T2 bench.py --gpus $N --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 1 --workload $WL > $OUT/ours_${WL}_n${N}_s$SP.json 2> $OUT/ours_${WL}_n${N}_s$SP.err
      echo "n$N $WL split=$SP $(python scripts/show_bench.py $OUT/ours_${WL}_n${N}_s$SP.json)" >> $OUT/sweep.txt
    done
  done
done
echo done > $OUT/DONE
