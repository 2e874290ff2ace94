#!/bin/bash
# bash scripts/gpu_ii2.sh TAG : parity of the split-mode paths (lean cross instantiation), then
# cfg2ii at N=2 over split cap x lean
TAG=${1:-ii2}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -p no:cacheprovider -k "split or ii or gd" > $OUT/pytest_multi.log 2>&1; echo "rc=$?" >> $OUT/pytest_multi.log
T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534"
for REP in 1 2; do
for E in "RP_XGPU_SPLIT=148" "RP_XGPU_SPLIT=296" "RP_XGPU_SPLIT=222" "RP_XGPU_SPLIT=296 RP_XGPU_LEAN=0" "RP_XGPU_SPLIT=74"; do
  env $E timeout 200 $T2 bench.py --gpus 2 --workload cfg2ii --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 1 > $OUT/t.json 2> $OUT/t.err
  echo "$E $(python scripts/show_bench.py $OUT/t.json)" >> $OUT/sweep.txt
done
done
echo done > $OUT/DONE
