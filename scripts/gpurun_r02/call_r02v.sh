# round 2, call v (4 GPUs): chunk-major dynamic claiming across a GPU's groups
export RP_WATCHDOG_S=60
OUT=gpurun_out/r02v; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_emulated.py -m gpu -x -q -p no:cacheprovider > $OUT/pytest_emul.log 2>&1; echo "rc=$?" >> $OUT/pytest_emul.log
grep -q "rc=0" $OUT/pytest_emul.log || exit 1
timeout 1200 python -m pytest tests/test_gpu_multi.py -m gpu -x -q -p no:cacheprovider -k "parity and not nvls or native" > $OUT/pytest_multi.log 2>&1; echo "rc=$?" >> $OUT/pytest_multi.log
grep -q "rc=0" $OUT/pytest_multi.log || exit 1
T4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29581"
T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29582"
timeout 900 $T4 bench.py --gpus 4 > $OUT/default_n4.json 2> $OUT/default_n4.err
RP_XGPU_DYN=0 timeout 600 $T4 bench.py --gpus 4 --no-extras > $OUT/default_n4_dyn0.json 2> $OUT/default_n4_dyn0.err
timeout 900 $T2 bench.py --gpus 2 > $OUT/default_n2.json 2> $OUT/default_n2.err
for wl in cfg3 cfg4; do
  timeout 300 $T4 bench.py --gpus 4 --workload $wl --steps 100 --e2e-steps 2 --no-extras > $OUT/ours_${wl}_n4.json 2> $OUT/ours_${wl}_n4.err
  RP_XGPU_DYN=0 timeout 300 $T4 bench.py --gpus 4 --workload $wl --steps 100 --e2e-steps 2 --no-extras > $OUT/ours_${wl}_n4_dyn0.json 2> $OUT/ours_${wl}_n4_dyn0.err
done
