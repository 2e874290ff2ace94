# round 2, call x (2 GPUs): final driver tiers -- smoke(), pytest -m gpu (1 GPU visible), bench N=1 / reference / N=2
OUT=gpurun_out/r02x; mkdir -p $OUT
CUDA_VISIBLE_DEVICES=0 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
CUDA_VISIBLE_DEVICES=0 timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu_1gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu_1gpu.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > $OUT/bench_n1.json 2> $OUT/bench_n1.err
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/reference_n1.json 2> $OUT/reference_n1.err
T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29595"
timeout 900 $T2 bench.py --gpus 2 > $OUT/bench_n2.json 2> $OUT/bench_n2.err
timeout 300 $T2 bench.py --gpus 2 --impl reference --steps 3 --warmup 3 > $OUT/reference_n2.json 2> $OUT/reference_n2.err
