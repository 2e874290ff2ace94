#!/bin/bash
# bash scripts/gpu_4_final5.sh TAG : final 4-GPU confirmation of the round-1 build
TAG=${1:-f05}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider -k "native or split or bf16" > $OUT/pytest_multi.log 2>&1; echo "rc=$?" >> $OUT/pytest_multi.log
for NG in 2 4; do
  T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29534"
  timeout 300 $T2 bench.py --gpus $NG > $OUT/ours_default_n$NG.json 2> $OUT/ours_default_n$NG.err
done
T4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534"
timeout 300 $T4 bench.py --gpus 4 --impl nccl --steps 100 --warmup 5 > $OUT/nccl_default_n4.json 2> $OUT/nccl_default_n4.err
timeout 300 $T4 bench.py --gpus 4 --impl reference --steps 3 --warmup 3 > $OUT/reference_default_n4.json 2> $OUT/reference_default_n4.err
for WL in cfg2iibf16 cfg3 cfg4; do
  timeout 300 $T4 bench.py --gpus 4 --steps 100 --warmup 5 --workload $WL --no-cpu-baseline --e2e-steps 2 > $OUT/ours_${WL}_n4.json 2> $OUT/ours_${WL}_n4.err
done
echo done > $OUT/DONE
