#!/bin/bash
# bash scripts/gpu_4_final4.sh TAG : 4-GPU box: 1-GPU kernel + parity tests, multi-GPU native/split/bf16
# parity, then the default bench at N = 1, 2, 4 and cfg3 / cfg4 / bf16 Inter-Intra at N = 4
TAG=${1:-f04}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_engine.py -q -p no:cacheprovider > $OUT/pytest_1gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_1gpu.log
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider -k "native or split or bf16 or ii" > $OUT/pytest_multi.log 2>&1; echo "rc=$?" >> $OUT/pytest_multi.log
timeout 300 python bench.py --no-cpu-baseline > $OUT/ours_default_n1.json 2> $OUT/ours_default_n1.err
for NG in 2 4; do
  T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29534"
  timeout 300 $T2 bench.py --gpus $NG > $OUT/ours_default_n$NG.json 2> $OUT/ours_default_n$NG.err
done
T4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534"
for WL in cfg3 cfg2iibf16 cfg4; do
  timeout 300 $T4 bench.py --gpus 4 --steps 100 --warmup 5 --workload $WL --no-cpu-baseline --e2e-steps 2 > $OUT/ours_${WL}_n4.json 2> $OUT/ours_${WL}_n4.err
done
timeout 300 $T4 bench.py --gpus 4 > $OUT/ours_default_n4_rep.json 2> $OUT/ours_default_n4_rep.err
echo done > $OUT/DONE
