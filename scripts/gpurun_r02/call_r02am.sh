# round 2, call am (4 GPUs): chunk floor 2 per lane -- parity (emulated suite, 2/4-GPU native + poisoned
# cases), then the default N = 2 / N = 4 lines
OUT=gpurun_out/r02am; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_emulated.py -m gpu -q -x -p no:cacheprovider -k "not variant" > $OUT/pytest_emul.log 2>&1; echo "rc=$?" >> $OUT/pytest_emul.log
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -x -p no:cacheprovider -k "native or poison or knobs" > $OUT/pytest_multi.log 2>&1; echo "rc=$?" >> $OUT/pytest_multi.log
T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29595"
T4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29596"
timeout 600 $T2 bench.py --gpus 2 --no-extras > $OUT/bench_n2.json 2> $OUT/bench_n2.err
timeout 600 $T4 bench.py --gpus 4 > $OUT/bench_n4.json 2> $OUT/bench_n4.err
