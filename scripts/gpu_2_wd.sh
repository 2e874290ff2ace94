#!/bin/bash
# bash scripts/gpu_2_wd.sh TAG : 2-GPU check of the flag-wait watchdog (parity + default bench)
TAG=${1:-wd}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 420 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider > $OUT/pytest_multi.log 2>&1; echo "rc=$?" >> $OUT/pytest_multi.log
T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534"
timeout 240 $T2 bench.py --gpus 2 > $OUT/ours_default_n2.json 2> $OUT/ours_default_n2.err
timeout 240 $T2 bench.py --gpus 2 --steps 100 --warmup 5 --workload cfg3 --no-cpu-baseline --e2e-steps 2 > $OUT/ours_cfg3_n2.json 2> $OUT/ours_cfg3_n2.err
echo done > $OUT/DONE
