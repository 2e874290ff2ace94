#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, ncu launch list + full capture of the top kernel.
# Usage (from the repo root on the GPU box): bash scripts/gpu_check.sh [tag]
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -c "import torch;print(torch.cuda.get_device_name(0), torch.cuda.get_device_properties(0))" > $OUT/device.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py --steps 50 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 300 python bench.py --workload cfg1 --steps 100 --warmup 5 --no-cpu-baseline > $OUT/bench_cfg1.json 2> $OUT/bench_cfg1.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
CMD="python bench.py --steps 8 --warmup 3 --no-cpu-baseline --e2e-steps 1"
if timeout 300 $CMD > $OUT/ncu_plain.log 2>&1; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:preduce_ -s 6 -c 2 -o $OUT/prof $CMD > $OUT/ncu_full.log 2>&1
fi
echo done > $OUT/DONE
