#!/bin/bash
# bash scripts/gpu_var.sh TAG : split-mode parity, then run-to-run variance of cfg2ii at N=2 under
# the split-launch settings (tiles per CTA of the intra-GPU launch, cross-stream priority)
TAG=${1:-v1}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -p no:cacheprovider -k "split or ii or native" > $OUT/pytest_multi.log 2>&1; echo "rc=$?" >> $OUT/pytest_multi.log
RP_DYN_TPC=7 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "native or cfg2" > $OUT/pytest_tpc.log 2>&1; echo "rc=$?" >> $OUT/pytest_tpc.log
T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534"
for REP in 1 2 3 4; do
  for E in "RP_DYN_TPC=32" "RP_DYN_TPC=0 RP_XS_PRIO=0" "RP_DYN_TPC=8" "RP_DYN_TPC=128"; do
    env $E timeout 200 $T2 bench.py --gpus 2 --workload cfg2ii --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 1 > $OUT/t.json 2> $OUT/t.err
    echo "$E r$REP $(python scripts/show_bench.py $OUT/t.json)" >> $OUT/sweep.txt
  done
done
echo done > $OUT/DONE
