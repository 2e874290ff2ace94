# round 2, call r (1 GPU): the driver's GPU tier as it will run it -- smoke() + pytest -m gpu; default bench N=1
OUT=gpurun_out/r02r; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py > $OUT/bench_n1.json 2> $OUT/bench_n1.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/reference_n1.json 2> $OUT/reference_n1.err
timeout 300 python bench.py --workload cfg1 --steps 1000 --no-cpu-baseline > $OUT/cfg1.json 2> $OUT/cfg1.err
timeout 300 python bench.py --workload cfg2bf16 --no-cpu-baseline > $OUT/cfg2bf16.json 2> $OUT/cfg2bf16.err
