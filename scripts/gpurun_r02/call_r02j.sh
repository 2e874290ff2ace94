# round 2, call j (4 GPUs): parity at 4 GPUs; bench default N=4 with extras; configs[2]/[3] shapes; kp=3 xall on 3 GPUs; NVLS
export RP_WATCHDOG_S=60
OUT=gpurun_out/r02j; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_multi.py -m gpu -x -q -p no:cacheprovider -k "not async" > $OUT/pytest_multi.log 2>&1; echo "rc=$?" >> $OUT/pytest_multi.log
T4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29551"
T3="python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29552"
timeout 900 $T4 bench.py --gpus 4 > $OUT/default_n4.json 2> $OUT/default_n4.err
for wl in cfg3 cfg4 cfg4p4 xall xall_vgg cfg2ii; do
  timeout 300 $T4 bench.py --gpus 4 --workload $wl --steps 60 --e2e-steps 1 --no-extras > $OUT/ours_${wl}_n4.json 2> $OUT/ours_${wl}_n4.err
  timeout 300 $T4 bench.py --gpus 4 --workload $wl --impl nccl --steps 60 > $OUT/ar_${wl}_n4.json 2> $OUT/ar_${wl}_n4.err
done
timeout 300 $T4 bench.py --gpus 4 --workload cfg3 --impl nccl-group --steps 60 > $OUT/grp_cfg3_n4.json 2> $OUT/grp_cfg3_n4.err
timeout 300 $T4 bench.py --gpus 4 --workload cfg4 --impl nccl-group --steps 30 > $OUT/grp_cfg4_n4.json 2> $OUT/grp_cfg4_n4.err
for nv in 3 4; do timeout 300 $T4 bench.py --gpus 4 --workload xall --nvls $nv --steps 60 --e2e-steps 1 --no-extras > $OUT/nvls${nv}_xall_n4.json 2> $OUT/nvls${nv}_xall_n4.err; done
timeout 300 $T4 bench.py --gpus 4 --workload cfg3 --nvls 3 --steps 60 --e2e-steps 1 --no-extras > $OUT/nvls3_cfg3_n4.json 2> $OUT/nvls3_cfg3_n4.err
for wl in xall xall_vgg; do
  timeout 300 $T3 bench.py --gpus 3 --workload $wl --steps 60 --e2e-steps 1 --no-extras > $OUT/ours_${wl}_n3.json 2> $OUT/ours_${wl}_n3.err
  timeout 300 $T3 bench.py --gpus 3 --workload $wl --impl nccl --steps 60 > $OUT/ar_${wl}_n3.json 2> $OUT/ar_${wl}_n3.err
done
timeout 300 $T4 bench.py --gpus 4 --workload cfg5static --steps 30 --no-extras > $OUT/cfg5static_n4.json 2> $OUT/cfg5static_n4.err
timeout 300 $T4 bench.py --gpus 4 --workload cfg5static --impl nccl --steps 30 > $OUT/cfg5static_ar_n4.json 2> $OUT/cfg5static_ar_n4.err
