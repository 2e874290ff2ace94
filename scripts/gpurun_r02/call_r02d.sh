# round 2, call d (2 GPUs): release-only flags + 2 iterations per lane; parity; bench with extras
export RP_WATCHDOG_S=30
OUT=gpurun_out/r02d; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_emulated.py -m gpu -x -q -p no:cacheprovider > $OUT/pytest_emul.log 2>&1; echo "rc=$?" >> $OUT/pytest_emul.log
timeout 600 python -m pytest tests/test_gpu_multi.py -m gpu -x -q -p no:cacheprovider -k "parity and not nvls and not async" > $OUT/pytest_multi.log 2>&1; echo "rc=$?" >> $OUT/pytest_multi.log
python scripts/nvml_nvlink_probe.py > $OUT/nvml_probe.txt 2>&1
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29544"
timeout 900 $T bench.py --gpus 2 > $OUT/default_n2.json 2> $OUT/default_n2.err
for wl in cfg3 cfg4; do
RP_XGPU_PROFILE=$OUT/tl_$wl timeout 300 $T bench.py --gpus 2 --workload $wl --steps 20 --e2e-steps 1 > $OUT/tl_$wl.json 2>&1
python scripts/xgpu_timeline.py $OUT/tl_$wl.0 $OUT/tl_$wl.1 > $OUT/timeline_$wl.txt 2>&1
done
timeout 300 $T bench.py --gpus 2 --workload xall_vgg --steps 30 > $OUT/xall_vgg_n2.json 2> $OUT/xall_vgg_n2.err
timeout 300 $T bench.py --gpus 2 --workload cfg5static --steps 30 > $OUT/cfg5static_n2.json 2> $OUT/cfg5static_n2.err
timeout 300 $T bench.py --gpus 2 --workload cfg5static --impl nccl --steps 30 > $OUT/cfg5static_ar_n2.json 2> $OUT/cfg5static_ar_n2.err
timeout 300 $T bench.py --gpus 2 --workload cfg4p4 --steps 30 > $OUT/cfg4p4_n2.json 2> $OUT/cfg4p4_n2.err
