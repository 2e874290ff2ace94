# round 2, call g (2 GPUs): per-CTA wait breakdown of the cross kernel; nbuf / U sweep
export RP_WATCHDOG_S=30
OUT=gpurun_out/r02g; mkdir -p $OUT
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29547"
for wl in cfg4 xall_vgg xall_vgg_m2 xall; do
RP_XGPU_PROFILE=$OUT/tl_$wl timeout 300 $T bench.py --gpus 2 --workload $wl --steps 20 --e2e-steps 1 --no-extras > $OUT/tl_$wl.json 2>&1
python scripts/xgpu_timeline.py $OUT/tl_$wl.0 $OUT/tl_$wl.1 > $OUT/timeline_$wl.txt 2>&1
done
bash scripts/xgpu_sweep.sh r02g 2 "cfg4 xall_vgg_m2 xall" "RP_XGPU_NBUF=3;RP_XGPU_NBUF=2;RP_XGPU_NBUF=4;RP_XGPU_NBUF=6"
