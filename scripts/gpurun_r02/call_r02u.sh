# round 2, call u (4 GPUs): chunk count per lane >= 3 (ResNet-50 slices); default lines N = 4 and 2, cfg3/cfg4 at N = 4
export RP_WATCHDOG_S=60
OUT=gpurun_out/r02u; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -x -q -p no:cacheprovider -k "parity and not nvls" > $OUT/pytest_multi.log 2>&1; echo "rc=$?" >> $OUT/pytest_multi.log
T4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571"
T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29572"
timeout 900 $T4 bench.py --gpus 4 > $OUT/default_n4.json 2> $OUT/default_n4.err
timeout 900 $T2 bench.py --gpus 2 > $OUT/default_n2.json 2> $OUT/default_n2.err
for wl in cfg3 cfg4 xall; do
  timeout 300 $T4 bench.py --gpus 4 --workload $wl --steps 100 --e2e-steps 2 --no-extras > $OUT/ours_${wl}_n4.json 2> $OUT/ours_${wl}_n4.err
done
timeout 300 $T4 bench.py --gpus 4 --workload xall --impl nccl --steps 100 > $OUT/ar_xall_n4.json 2> $OUT/ar_xall_n4.err
