# round 2, call w (4 GPUs): claim order by schedule kind (part-major for static schedules)
export RP_WATCHDOG_S=60
OUT=gpurun_out/r02w; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_emulated.py -m gpu -x -q -p no:cacheprovider > $OUT/pytest_emul.log 2>&1; echo "rc=$?" >> $OUT/pytest_emul.log
grep -q "rc=0" $OUT/pytest_emul.log || exit 1
timeout 1200 python -m pytest tests/test_gpu_multi.py -m gpu -x -q -p no:cacheprovider -k "parity and not nvls or native" > $OUT/pytest_multi.log 2>&1; echo "rc=$?" >> $OUT/pytest_multi.log
grep -q "rc=0" $OUT/pytest_multi.log || exit 1
T4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29591"
timeout 900 $T4 bench.py --gpus 4 > $OUT/default_n4.json 2> $OUT/default_n4.err
for wl in cfg4 cfg4p4 cfg3 xall; do
  timeout 300 $T4 bench.py --gpus 4 --workload $wl --steps 100 --e2e-steps 2 --no-extras > $OUT/ours_${wl}_n4.json 2> $OUT/ours_${wl}_n4.err
done
RP_XGPU_CLAIM=chunk timeout 300 $T4 bench.py --gpus 4 --workload cfg4 --steps 100 --e2e-steps 2 --no-extras > $OUT/ours_cfg4_n4_chunk.json 2> $OUT/ours_cfg4_n4_chunk.err
RP_XGPU_CLAIM=part timeout 300 $T4 bench.py --gpus 4 --workload cfg3 --steps 100 --e2e-steps 2 --no-extras > $OUT/ours_cfg3_n4_part.json 2> $OUT/ours_cfg3_n4_part.err
