#!/bin/bash
# bash scripts/gpu_2_final6.sh TAG : 2-GPU confirmation of the final round-1 kernels (after 60ce049)
TAG=${1:-f06}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 420 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider -k "native or split or bf16" > $OUT/pytest_multi.log 2>&1; echo "rc=$?" >> $OUT/pytest_multi.log
T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534"
timeout 240 $T2 bench.py --gpus 2 > $OUT/ours_default_n2.json 2> $OUT/ours_default_n2.err
timeout 240 python bench.py > $OUT/ours_default_n1.json 2> $OUT/ours_default_n1.err
echo done > $OUT/DONE
