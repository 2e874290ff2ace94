#!/bin/bash
# bash scripts/gpu_native.sh TAG : native lockstep executor parity (1 and 2+ GPUs) and the
# per-call vs native bench comparison (1 GPU: cfg1, cfg2; N GPUs: cfg3, cfg2ii)
TAG=${1:-nx1}; OUT=gpurun_out/$TAG; mkdir -p $OUT
NG=$(nvidia-smi -L | wc -l)
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k native > $OUT/pytest_native.log 2>&1; echo "rc=$?" >> $OUT/pytest_native.log
timeout 600 python -m pytest tests/test_gpu_multi.py -q -x -p no:cacheprovider -k native > $OUT/pytest_multi_native.log 2>&1; echo "rc=$?" >> $OUT/pytest_multi_native.log
for M in "" "--per-call"; do
  for WL in cfg1 cfg2; do
    timeout 300 python bench.py --workload $WL --steps 200 --warmup 5 --no-cpu-baseline --e2e-steps 2 $M > $OUT/t.json 2>$OUT/t.err
    echo "n1 $WL $M $(python scripts/show_bench.py $OUT/t.json)" >> $OUT/sweep.txt
  done
done
T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29534"
for REP in 1 2 3; do
  for M in "" "--per-call"; do
    for WL in cfg3 cfg2ii; do
      timeout 200 $T2 bench.py --gpus $NG --workload $WL --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 1 $M > $OUT/t.json 2> $OUT/t.err
      echo "n$NG $WL $M r$REP $(python scripts/show_bench.py $OUT/t.json)" >> $OUT/sweep.txt
    done
  done
done
echo done > $OUT/DONE
