#!/bin/bash
# bash scripts/gpu_nvls.sh TAG : NVLS P-Reduce parity (2 and 4 GPUs) + 4-GPU benches vs the push kernel
TAG=${1:-nv4}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_multi.py -k nvls -q -p no:cacheprovider > $OUT/pytest_nvls.log 2>&1; echo "rc=$?" >> $OUT/pytest_nvls.log
T4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534"
T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535"
timeout 300 $T4 bench.py --gpus 4 --steps 100 --warmup 5 --workload cfg3 > $OUT/cfg3_n4_push.json 2> $OUT/cfg3_n4_push.err
for P in 0 25 50 75; do
  RP_NVLS_HBM_PCT=$P timeout 300 $T4 bench.py --gpus 4 --steps 100 --warmup 5 --workload cfg3 --nvls 3 > $OUT/cfg3_n4_nv3_p$P.json 2> $OUT/cfg3_n4_nv3_p$P.err
done
for P in 0 50; do
  RP_NVLS_HBM_PCT=$P timeout 300 $T2 bench.py --gpus 2 --steps 100 --warmup 5 --workload cfg3 --nvls 2 > $OUT/cfg3_n2_nv2_p$P.json 2> $OUT/cfg3_n2_nv2_p$P.err
  RP_NVLS_HBM_PCT=$P timeout 300 $T4 bench.py --gpus 4 --steps 100 --warmup 5 --workload cfg2 --nvls 3 > $OUT/cfg2_n4_nv3_p$P.json 2> $OUT/cfg2_n4_nv3_p$P.err
done
echo done > $OUT/DONE
