# round 2, call ag (4 GPUs): final confirmation at HEAD -- smoke(), pytest -m gpu (1 GPU visible),
# bench N=1 / reference, multi-GPU pytest (4 visible), bench N=2 / N=4 default lines
OUT=gpurun_out/r02ag; mkdir -p $OUT
CUDA_VISIBLE_DEVICES=0 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
CUDA_VISIBLE_DEVICES=0 timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu_1gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu_1gpu.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > $OUT/bench_n1.json 2> $OUT/bench_n1.err
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/reference_n1.json 2> $OUT/reference_n1.err
timeout 1200 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider > $OUT/pytest_multi_4gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_multi_4gpu.log
T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29595"
T4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29596"
timeout 900 $T2 bench.py --gpus 2 > $OUT/bench_n2.json 2> $OUT/bench_n2.err
timeout 900 $T4 bench.py --gpus 4 > $OUT/bench_n4.json 2> $OUT/bench_n4.err
