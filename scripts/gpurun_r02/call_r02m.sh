# round 2, call m (4 GPUs): kernels preloaded at rp_init (no lazy-loading stalls in timed regions)
export RP_WATCHDOG_S=60
OUT=gpurun_out/r02m; mkdir -p $OUT
T4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29554"
timeout 900 $T4 bench.py --gpus 4 > $OUT/default_n4.json 2> $OUT/default_n4.err
for wl in cfg3 cfg4 cfg4p4 xall xall_vgg cfg2ii; do
  RP_BENCH_DUMP_RECS=$OUT/recs_${wl}.json timeout 300 $T4 bench.py --gpus 4 --workload $wl --steps 100 --e2e-steps 2 --no-extras > $OUT/ours_${wl}_n4.json 2> $OUT/ours_${wl}_n4.err
done
for wl in cfg3 cfg4p4; do
  timeout 300 $T4 bench.py --gpus 4 --workload $wl --impl nccl --steps 100 > $OUT/ar_${wl}_n4.json 2> $OUT/ar_${wl}_n4.err
  timeout 300 $T4 bench.py --gpus 4 --workload $wl --impl nccl-group --steps 60 > $OUT/grp_${wl}_n4.json 2> $OUT/grp_${wl}_n4.err
done
