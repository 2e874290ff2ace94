#!/bin/bash
# bash scripts/gpu_2_wd2.sh TAG : repeat the default N=2 bench 3x (watchdog build variance)
TAG=${1:-wd2}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534"
for i in 1 2 3; do
  timeout 200 $T2 bench.py --gpus 2 --no-cpu-baseline --e2e-steps 2 > $OUT/ours_default_n2_$i.json 2> $OUT/ours_default_n2_$i.err
done
echo done > $OUT/DONE
