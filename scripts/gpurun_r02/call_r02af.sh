# round 2, call af (4 GPUs): early A flags (RP_XGPU_EARLY_A=1) -- parity (emulated + 2/4 GPUs), then A/B sweeps
OUT=gpurun_out/r02af; mkdir -p $OUT
RP_XGPU_EARLY_A=1 timeout 600 python -m pytest tests/test_gpu_emulated.py -m gpu -q -x -p no:cacheprovider > $OUT/pytest_emul.log 2>&1; echo "rc=$?" >> $OUT/pytest_emul.log
RP_XGPU_EARLY_A=1 timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -x -p no:cacheprovider -k "native or poison" > $OUT/pytest_multi.log 2>&1; echo "rc=$?" >> $OUT/pytest_multi.log
bash scripts/xgpu_sweep.sh r02af 2 "r50x8 cfg4 cfg3 xall" "RP_XGPU_EARLY_A=0;RP_XGPU_EARLY_A=1;RP_XGPU_EARLY_A=0;RP_XGPU_EARLY_A=1"
mv $OUT/sweep.txt $OUT/sweep2.txt
bash scripts/xgpu_sweep.sh r02af 4 "r50x8 cfg4 cfg3 xall" "RP_XGPU_EARLY_A=0;RP_XGPU_EARLY_A=1;RP_XGPU_EARLY_A=0;RP_XGPU_EARLY_A=1"
mv $OUT/sweep.txt $OUT/sweep4.txt
