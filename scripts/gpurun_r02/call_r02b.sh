# round 2, call b (2 GPUs): new lane-pipelined cross-GPU kernel -- emulated + real parity, bench
export RP_WATCHDOG_S=20
OUT=gpurun_out/r02b; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 900 python -m pytest tests/test_gpu_emulated.py -m gpu -x -q -p no:cacheprovider > $OUT/pytest_emul.log 2>&1; echo "rc=$?" >> $OUT/pytest_emul.log
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -x -q -p no:cacheprovider -k "not nvls and not async" > $OUT/pytest_multi.log 2>&1; echo "rc=$?" >> $OUT/pytest_multi.log
bash scripts/gpu_multi.sh r02b 2 "cfg4 cfg3 r50x8"
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29542"
for wl in cfg4 r50x8 cfg3; do
RP_XGPU_PROFILE=$OUT/tl_$wl timeout 300 $T bench.py --gpus 2 --workload $wl --steps 20 --e2e-steps 1 > $OUT/tl_$wl.json 2>&1
python scripts/xgpu_timeline.py $OUT/tl_$wl.0 $OUT/tl_$wl.1 > $OUT/timeline_$wl.txt 2>&1
done
python scripts/nvml_nvlink_probe.py > $OUT/nvml_probe.txt 2>&1
