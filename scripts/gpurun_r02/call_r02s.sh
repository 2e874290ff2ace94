# round 2, call s (2 GPUs): dynamic chunk claiming in the ws kernel: parity, dyn on/off sweep, CTA end spread
export RP_WATCHDOG_S=30
OUT=gpurun_out/r02s; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_emulated.py -m gpu -x -q -p no:cacheprovider > $OUT/pytest_emul.log 2>&1; echo "rc=$?" >> $OUT/pytest_emul.log
grep -q "rc=0" $OUT/pytest_emul.log || exit 1
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -x -q -p no:cacheprovider -k "not nvls and not async" > $OUT/pytest_multi.log 2>&1; echo "rc=$?" >> $OUT/pytest_multi.log
grep -q "rc=0" $OUT/pytest_multi.log || exit 1
bash scripts/xgpu_sweep.sh r02s 2 "xall cfg3 cfg4 r50x8 xall_vgg" "RP_XGPU_DYN=1;RP_XGPU_DYN=0;RP_XGPU_DYN=1 RP_XGPU_ITERS=6;RP_XGPU_DYN=1 RP_XGPU_BLAG=2"
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29557"
for wl in xall cfg4; do
RP_XGPU_PROFILE=$OUT/tl_$wl timeout 300 $T bench.py --gpus 2 --workload $wl --steps 20 --e2e-steps 1 --no-extras > $OUT/tl_$wl.json 2>&1
python scripts/xgpu_timeline.py $OUT/tl_$wl.0 $OUT/tl_$wl.1 > $OUT/timeline_$wl.txt 2>&1
done
