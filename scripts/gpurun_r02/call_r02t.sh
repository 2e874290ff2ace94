# round 2, call t (4 GPUs): final multi-GPU parity + the round's multi-GPU bench lines (N = 2, 3, 4)
export RP_WATCHDOG_S=60
OUT=gpurun_out/r02t; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider > $OUT/pytest_multi.log 2>&1; echo "rc=$?" >> $OUT/pytest_multi.log
T4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561"
T3="python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29562"
T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29563"
timeout 900 $T4 bench.py --gpus 4 > $OUT/default_n4.json 2> $OUT/default_n4.err
timeout 900 $T2 bench.py --gpus 2 > $OUT/default_n2.json 2> $OUT/default_n2.err
for wl in cfg3 cfg4 cfg4p4 xall xall_vgg cfg2ii cfg2iibf16; do
  timeout 300 $T4 bench.py --gpus 4 --workload $wl --steps 100 --e2e-steps 2 --no-extras > $OUT/ours_${wl}_n4.json 2> $OUT/ours_${wl}_n4.err
done
for wl in cfg3 cfg4 cfg4p4 xall xall_vgg cfg2ii; do
  timeout 300 $T4 bench.py --gpus 4 --workload $wl --impl nccl --steps 100 > $OUT/ar_${wl}_n4.json 2> $OUT/ar_${wl}_n4.err
done
for wl in cfg3 cfg4 cfg4p4; do
  timeout 300 $T4 bench.py --gpus 4 --workload $wl --impl nccl-group --steps 60 > $OUT/grp_${wl}_n4.json 2> $OUT/grp_${wl}_n4.err
done
for wl in xall xall_vgg; do
  timeout 300 $T3 bench.py --gpus 3 --workload $wl --steps 100 --e2e-steps 2 --no-extras > $OUT/ours_${wl}_n3.json 2> $OUT/ours_${wl}_n3.err
  timeout 300 $T3 bench.py --gpus 3 --workload $wl --impl nccl --steps 100 > $OUT/ar_${wl}_n3.json 2> $OUT/ar_${wl}_n3.err
done
timeout 300 $T4 bench.py --gpus 4 --workload cfg5static --steps 30 --no-extras > $OUT/ours_cfg5static_n4.json 2> $OUT/ours_cfg5static_n4.err
timeout 300 $T4 bench.py --gpus 4 --workload cfg5static --impl nccl --steps 30 > $OUT/ar_cfg5static_n4.json 2> $OUT/ar_cfg5static_n4.err
for s in 0 5; do
  timeout 300 $T4 bench.py --gpus 4 --workload cfg5 --slow $s > $OUT/ours_cfg5_s${s}_n4.json 2> $OUT/ours_cfg5_s${s}_n4.err
  timeout 300 $T4 bench.py --gpus 4 --workload cfg5 --slow $s --impl nccl --steps 30 > $OUT/ar_cfg5_s${s}_n4.json 2> $OUT/ar_cfg5_s${s}_n4.err
done
timeout 300 $T4 bench.py --gpus 4 --workload xall --nvls 4 --steps 60 --e2e-steps 1 --no-extras > $OUT/nvls4_xall_n4.json 2> $OUT/nvls4_xall_n4.err
timeout 300 $T4 bench.py --gpus 4 --workload xall_vgg --nvls 4 --steps 60 --e2e-steps 1 --no-extras > $OUT/nvls4_xall_vgg_n4.json 2> $OUT/nvls4_xall_vgg_n4.err
