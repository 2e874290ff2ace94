#!/bin/bash
# bash scripts/gpu_4_final7.sh TAG : 4-GPU confirmation of the final round-1 kernels (after 60ce049)
TAG=${1:-f07}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider -k "native or split or bf16" > $OUT/pytest_multi.log 2>&1; echo "rc=$?" >> $OUT/pytest_multi.log
T4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534"
timeout 150 $T4 bench.py --gpus 4 > $OUT/ours_default_n4.json 2> $OUT/ours_default_n4.err
timeout 120 $T4 bench.py --gpus 4 --steps 100 --warmup 5 --workload cfg2iibf16 --no-cpu-baseline --e2e-steps 2 > $OUT/ours_cfg2iibf16_n4.json 2> $OUT/ours_cfg2iibf16_n4.err
echo done > $OUT/DONE
