# round 2, call f (2 GPUs): new parity tests; split-order sweep on the HBM+NVLink workloads
export RP_WATCHDOG_S=30
OUT=gpurun_out/r02f; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_emulated.py tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider > $OUT/pytest_1gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_1gpu.log
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -x -q -p no:cacheprovider -k "native or split or geometry" > $OUT/pytest_multi.log 2>&1; echo "rc=$?" >> $OUT/pytest_multi.log
bash scripts/xgpu_sweep.sh r02f 2 "cfg4 r50x8 cfg2ii" "RP_SPLIT_ORDER=0;RP_SPLIT_ORDER=1;RP_SPLIT_ORDER=2;RP_XGPU_SPLIT=148;RP_XGPU_SPLIT=222"
