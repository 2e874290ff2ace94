# round 2, call l (4 GPUs): fused L jobs + BLAG 3 at N=4: bench default (extras), configs[2]/[3] shapes, cfg3 diagnosis
export RP_WATCHDOG_S=60
OUT=gpurun_out/r02l; mkdir -p $OUT
T4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29553"
timeout 600 python -m pytest tests/test_gpu_multi.py -m gpu -x -q -p no:cacheprovider -k "parity and not nvls" > $OUT/pytest_multi.log 2>&1; echo "rc=$?" >> $OUT/pytest_multi.log
timeout 900 $T4 bench.py --gpus 4 > $OUT/default_n4.json 2> $OUT/default_n4.err
for wl in cfg3 cfg4 cfg4p4 xall; do
  timeout 300 $T4 bench.py --gpus 4 --workload $wl --steps 60 --e2e-steps 1 --no-extras > $OUT/ours_${wl}_n4.json 2> $OUT/ours_${wl}_n4.err
done
RP_BENCH_DUMP_RECS=$OUT/recs_cfg3.json RP_XGPU_PROFILE=$OUT/tl_cfg3 timeout 300 $T4 bench.py --gpus 4 --workload cfg3 --steps 20 --e2e-steps 1 --no-extras > $OUT/tl_cfg3.json 2>&1
python scripts/xgpu_timeline.py $OUT/tl_cfg3.0 $OUT/tl_cfg3.1 $OUT/tl_cfg3.2 $OUT/tl_cfg3.3 > $OUT/timeline_cfg3.txt 2>&1
RP_BENCH_DUMP_RECS=$OUT/recs_xall.json timeout 300 $T4 bench.py --gpus 4 --workload xall --steps 20 --e2e-steps 1 --no-extras > $OUT/recs_xall_bench.json 2>&1
timeout 300 $T4 bench.py --gpus 4 --workload cfg3 --impl nccl-group --steps 60 > $OUT/grp_cfg3_n4.json 2> $OUT/grp_cfg3_n4.err
