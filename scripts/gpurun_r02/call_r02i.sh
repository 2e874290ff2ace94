# round 2, call i (2 GPUs): bulk-store granularity probe; B-lag / iterations sweep of the ws kernel
export RP_WATCHDOG_S=30
OUT=gpurun_out/r02i; mkdir -p $OUT
PROBE_ONLY_SPLIT=1 timeout 120 ./build/bulk_push_probe > $OUT/bulk_push_granularity.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_emulated.py -m gpu -x -q -p no:cacheprovider > $OUT/pytest_emul.log 2>&1; echo "rc=$?" >> $OUT/pytest_emul.log
RP_XGPU_BLAG=3 timeout 300 python -m pytest tests/test_gpu_emulated.py -m gpu -x -q -p no:cacheprovider > $OUT/pytest_emul_blag3.log 2>&1; echo "rc=$?" >> $OUT/pytest_emul_blag3.log
bash scripts/xgpu_sweep.sh r02i 2 "cfg4 xall_vgg xall r50x8" "RP_XGPU_BLAG=2;RP_XGPU_BLAG=3;RP_XGPU_BLAG=3 RP_XGPU_ITERS=6;RP_XGPU_BLAG=4 RP_XGPU_ITERS=8"
