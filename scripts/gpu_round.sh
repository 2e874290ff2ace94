#!/bin/bash
# One gpurun call (any GPU count): full GPU suite, smoke, 1-GPU bench (default = configs[1]) +
# cfg1 + bf16 + reference arm, ncu launch list + full capture of the top kernel, then the
# default multi-GPU bench (and plain-GD cfg2 + the NCCL all-reduce baseline) at every N <= GPUs.
TAG=${1:-r01f}
OUT=gpurun_out/$TAG
mkdir -p $OUT
NG=$(nvidia-smi -L | wc -l)
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 300 python bench.py --workload cfg1 --steps 100 --warmup 5 --no-cpu-baseline > $OUT/bench_cfg1.json 2> $OUT/bench_cfg1.err
timeout 300 python bench.py --workload cfg2bf16 --no-cpu-baseline > $OUT/bench_cfg2bf16.json 2> $OUT/bench_cfg2bf16.err
timeout 300 python bench.py --workload cfg2ii --no-cpu-baseline > $OUT/bench_cfg2ii.json 2> $OUT/bench_cfg2ii.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
CMD="python bench.py --steps 8 --warmup 3 --no-cpu-baseline --e2e-steps 1"
if timeout 300 $CMD > $OUT/ncu_plain.log 2>&1; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:preduce_ -s 6 -c 2 -o $OUT/prof $CMD > $OUT/ncu_full.log 2>&1
fi
for N in 2 4 8; do
  [ $N -gt $NG ] && continue
  T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29534"
  timeout 400 $T2 bench.py --gpus $N > $OUT/ours_default_n$N.json 2> $OUT/ours_default_n$N.err
  timeout 300 $T2 bench.py --gpus $N --impl nccl --steps 100 --warmup 5 > $OUT/nccl_default_n$N.json 2> $OUT/nccl_default_n$N.err
  timeout 300 $T2 bench.py --gpus $N --workload cfg2 --steps 100 --warmup 5 --no-cpu-baseline > $OUT/ours_cfg2_n$N.json 2> $OUT/ours_cfg2_n$N.err
  timeout 300 $T2 bench.py --gpus $N --impl reference --steps 3 --warmup 3 > $OUT/reference_default_n$N.json 2> $OUT/reference_default_n$N.err
done
echo done > $OUT/DONE
