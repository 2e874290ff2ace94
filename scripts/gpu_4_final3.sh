#!/bin/bash
# bash scripts/gpu_4_final3.sh TAG : 4-GPU box: native-executor + split + bf16 multi-GPU parity, then
# the default bench (N = 2, 4) vs NCCL all-reduce, reference arm, and the other multi-GPU workloads
TAG=${1:-f03}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider -k "native or split or bf16" > $OUT/pytest_multi.log 2>&1; echo "rc=$?" >> $OUT/pytest_multi.log
for NG in 2 4; do
  T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29534"
  timeout 300 $T2 bench.py --gpus $NG > $OUT/ours_default_n$NG.json 2> $OUT/ours_default_n$NG.err
  timeout 300 $T2 bench.py --gpus $NG --impl nccl --steps 100 --warmup 5 > $OUT/nccl_default_n$NG.json 2> $OUT/nccl_default_n$NG.err
  timeout 300 $T2 bench.py --gpus $NG --impl reference --steps 3 --warmup 3 > $OUT/reference_default_n$NG.json 2> $OUT/reference_default_n$NG.err
  for WL in cfg3 cfg4 cfg2 cfg2iibf16 xall xall_vgg; do
    timeout 300 $T2 bench.py --gpus $NG --steps 100 --warmup 5 --workload $WL --no-cpu-baseline --e2e-steps 2 > $OUT/ours_${WL}_n$NG.json 2> $OUT/ours_${WL}_n$NG.err
  done
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 4 > $OUT/ours_default_n4_rep.json 2> $OUT/ours_default_n4_rep.err
echo done > $OUT/DONE
