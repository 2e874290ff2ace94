# round 2, call al (4 GPUs): ITERS 3 (default) vs 2 at ResNet-50 size, N = 4, alternated three times
OUT=gpurun_out/r02al; mkdir -p $OUT
bash scripts/xgpu_sweep.sh r02al 4 "cfg3 r50x8" "RP_XGPU_ITERS=0;RP_XGPU_ITERS=2;RP_XGPU_ITERS=0;RP_XGPU_ITERS=2;RP_XGPU_ITERS=0;RP_XGPU_ITERS=2"
