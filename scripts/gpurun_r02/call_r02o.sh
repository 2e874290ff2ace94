# round 2, call o (2 GPUs): two SIGs per lane iteration (A flags at the end of their own iteration)
export RP_WATCHDOG_S=30
OUT=gpurun_out/r02o; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_emulated.py -m gpu -x -q -p no:cacheprovider > $OUT/pytest_emul.log 2>&1; echo "rc=$?" >> $OUT/pytest_emul.log
grep -q "rc=0" $OUT/pytest_emul.log || exit 1
RP_XGPU_BLAG=2 timeout 600 python -m pytest tests/test_gpu_emulated.py -m gpu -x -q -p no:cacheprovider > $OUT/pytest_emul_bl2.log 2>&1; echo "rc=$?" >> $OUT/pytest_emul_bl2.log
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -x -q -p no:cacheprovider -k "parity and not nvls" > $OUT/pytest_multi.log 2>&1; echo "rc=$?" >> $OUT/pytest_multi.log
grep -q "rc=0" $OUT/pytest_multi.log || exit 1
bash scripts/xgpu_sweep.sh r02o 2 "xall cfg3 cfg4 r50x8 xall_vgg" "RP_XGPU_SIG2=1 RP_XGPU_BLAG=1;RP_XGPU_SIG2=1 RP_XGPU_BLAG=2;RP_XGPU_SIG2=1 RP_XGPU_BLAG=1 RP_XGPU_ITERS=4;RP_XGPU_SIG2=0 RP_XGPU_BLAG=3"
