# round 2, call q (2 GPUs): compute-sanitizer racecheck (1 GPU, one tool per call); per-CTA begin/end timelines
OUT=gpurun_out/r02q; mkdir -p $OUT
bash scripts/call_r02_san_racecheck.sh
export RP_WATCHDOG_S=30
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29556"
for wl in xall xall_vgg cfg4; do
RP_XGPU_PROFILE=$OUT/tl_$wl timeout 300 $T bench.py --gpus 2 --workload $wl --steps 20 --e2e-steps 1 --no-extras > $OUT/tl_$wl.json 2>&1
python scripts/xgpu_timeline.py $OUT/tl_$wl.0 $OUT/tl_$wl.1 > $OUT/timeline_$wl.txt 2>&1
done
