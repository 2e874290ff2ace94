#!/bin/bash
# bash scripts/gpu_1_final8.sh TAG : the round-end 1-GPU sequence (build, smoke, pytest -m gpu, bench)
TAG=${1:-f08}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 200 python bench.py > $OUT/bench.json 2> $OUT/bench.err
echo done > $OUT/DONE
