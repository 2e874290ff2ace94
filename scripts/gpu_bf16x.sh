#!/bin/bash
# bash scripts/gpu_bf16x.sh TAG : cross-GPU bf16 parity + bf16 multi-GPU benches
TAG=${1:-bx1}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider -k "bf16 or split" > $OUT/pytest_multi.log 2>&1; echo "rc=$?" >> $OUT/pytest_multi.log
NG=$(nvidia-smi -L | wc -l)
for N in 2 4; do
  [ $N -gt $NG ] && continue
  T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29534"
  for WL in cfg2iibf16 cfg2bf16 cfg2ii; do
    timeout 200 $T2 bench.py --gpus $N --workload $WL --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 1 > $OUT/ours_${WL}_n$N.json 2> $OUT/ours_${WL}_n$N.err
    echo "n$N $WL $(python scripts/show_bench.py $OUT/ours_${WL}_n$N.json)" >> $OUT/sweep.txt
  done
done
echo done > $OUT/DONE
