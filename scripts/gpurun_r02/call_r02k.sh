# round 2, call k (2 GPUs): fused intra-GPU groups (L jobs) in the ws kernel: parity + fuse on/off; graph replay tests
export RP_WATCHDOG_S=30
OUT=gpurun_out/r02k; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_emulated.py tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider > $OUT/pytest_1gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_1gpu.log
grep -q "rc=0" $OUT/pytest_1gpu.log || exit 1
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -x -q -p no:cacheprovider -k "not nvls and not async" > $OUT/pytest_multi.log 2>&1; echo "rc=$?" >> $OUT/pytest_multi.log
grep -q "rc=0" $OUT/pytest_multi.log || exit 1
bash scripts/xgpu_sweep.sh r02k 2 "cfg4 r50x8 cfg2ii" "RP_XGPU_FUSE=1;RP_XGPU_FUSE=0"
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29549"
timeout 300 $T bench.py --gpus 2 --impl nccl-group --steps 60 > $OUT/grp_r50x8_n2.json 2> $OUT/grp_r50x8_n2.err
timeout 300 python bench.py --workload cfg1 --steps 500 --no-cpu-baseline > $OUT/cfg1_graph.json 2> $OUT/cfg1_graph.err
RP_XGPU_PROFILE=$OUT/tl_cfg4 timeout 300 $T bench.py --gpus 2 --workload cfg4 --steps 20 --e2e-steps 1 --no-extras > $OUT/tl_cfg4.json 2>&1
python scripts/xgpu_timeline.py $OUT/tl_cfg4.0 $OUT/tl_cfg4.1 > $OUT/timeline_cfg4.txt 2>&1
