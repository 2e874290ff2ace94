# round 2, call ah (4 GPUs): tail chunks carved out of the big chunks (RP_XGPU_TAIL_KEEP=1) at N = 4
OUT=gpurun_out/r02ah; mkdir -p $OUT
RP_XGPU_TAIL=296 RP_XGPU_TAIL_TILES=2 RP_XGPU_TAIL_KEEP=1 timeout 600 python -m pytest tests/test_gpu_emulated.py -m gpu -q -x -p no:cacheprovider > $OUT/pytest_emul.log 2>&1; echo "rc=$?" >> $OUT/pytest_emul.log
bash scripts/xgpu_sweep.sh r02ah 4 "cfg3 r50x8 xall cfg4" "RP_XGPU_TAIL=0;RP_XGPU_TAIL=296 RP_XGPU_TAIL_TILES=2 RP_XGPU_TAIL_KEEP=1;RP_XGPU_TAIL=296 RP_XGPU_TAIL_TILES=1 RP_XGPU_TAIL_KEEP=1;RP_XGPU_TAIL=592 RP_XGPU_TAIL_TILES=1 RP_XGPU_TAIL_KEEP=1"
