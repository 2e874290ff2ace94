#!/bin/bash
# bash scripts/gpu_chk2.sh TAG [WORKLOADS...] : re-measure workloads at N = 2 (and 4 if present)
TAG=${1:-k1}; shift; WLS=${@:-cfg4 cfg3 cfg2ii}
OUT=gpurun_out/$TAG; mkdir -p $OUT
NG=$(nvidia-smi -L | wc -l)
for N in 2 4; do
  [ $N -gt $NG ] && continue
  T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29534"
  for REP in 1 2; do
    for WL in $WLS; do
      timeout 200 $T2 bench.py --gpus $N --workload $WL --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 1 > $OUT/ours_${WL}_n${N}_r$REP.json 2> $OUT/ours_${WL}_n${N}_r$REP.err
      echo "n$N $WL r$REP $(python scripts/show_bench.py $OUT/ours_${WL}_n${N}_r$REP.json)" >> $OUT/sweep.txt
    done
  done
done
echo done > $OUT/DONE
