# round 2, call ak (4 GPUs): chunks per lane and B lag re-checked with early A flags, ResNet-50 size, N = 4
OUT=gpurun_out/r02ak; mkdir -p $OUT
bash scripts/xgpu_sweep.sh r02ak 4 "cfg3 r50x8 xall" "RP_XGPU_ITERS=0;RP_XGPU_ITERS=4;RP_XGPU_ITERS=2;RP_XGPU_BLAG=2"
