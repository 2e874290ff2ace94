# round 2, call y (2 GPUs): single-tile tail chunks; watchdog test
export RP_WATCHDOG_S=30
OUT=gpurun_out/r02y; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_emulated.py -m gpu -x -q -p no:cacheprovider > $OUT/pytest_emul.log 2>&1; echo "rc=$?" >> $OUT/pytest_emul.log
grep -q "rc=0" $OUT/pytest_emul.log || exit 1
timeout 1200 python -m pytest tests/test_gpu_multi.py -m gpu -x -q -p no:cacheprovider -k "parity and not nvls or native or geometry" > $OUT/pytest_multi.log 2>&1; echo "rc=$?" >> $OUT/pytest_multi.log
grep -q "rc=0" $OUT/pytest_multi.log || exit 1
unset RP_WATCHDOG_S
timeout 300 python -m pytest tests/test_gpu_multi.py -m gpu -x -q -p no:cacheprovider -k "watchdog" > $OUT/pytest_watchdog.log 2>&1; echo "rc=$?" >> $OUT/pytest_watchdog.log
export RP_WATCHDOG_S=30
bash scripts/xgpu_sweep.sh r02y 2 "xall cfg3 r50x8 cfg4 xall_vgg" "RP_XGPU_TAIL=296;RP_XGPU_TAIL=0;RP_XGPU_TAIL=592"
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29597"
RP_XGPU_PROFILE=$OUT/tl_xall timeout 300 $T bench.py --gpus 2 --workload xall --steps 20 --e2e-steps 1 --no-extras > $OUT/tl_xall.json 2>&1
python scripts/xgpu_timeline.py $OUT/tl_xall.0 $OUT/tl_xall.1 > $OUT/timeline_xall.txt 2>&1
