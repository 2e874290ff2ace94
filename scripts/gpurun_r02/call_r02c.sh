# round 2, call c (2 GPUs): bulk-store/signal probe; new bench.py (default N=1 and N=2 with extras)
export RP_WATCHDOG_S=30
OUT=gpurun_out/r02c; mkdir -p $OUT
timeout 300 ./build/bulk_push_probe > $OUT/bulk_push_probe.txt 2>&1
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29543"
timeout 600 $T bench.py --gpus 2 > $OUT/default_n2.json 2> $OUT/default_n2.err
timeout 300 python bench.py --cpu-budget 5 > $OUT/default_n1.json 2> $OUT/default_n1.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/reference_n1.json 2> $OUT/reference_n1.err
timeout 300 $T bench.py --gpus 2 --workload cfg5static --steps 30 --no-extras > $OUT/cfg5static_n2.json 2> $OUT/cfg5static_n2.err
timeout 300 $T bench.py --gpus 2 --workload cfg5static --impl nccl --steps 30 > $OUT/cfg5static_ar_n2.json 2> $OUT/cfg5static_ar_n2.err
timeout 300 $T bench.py --gpus 2 --workload cfg4p4 --steps 30 > $OUT/cfg4p4_n2.json 2> $OUT/cfg4p4_n2.err
