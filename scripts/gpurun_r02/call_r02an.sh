# round 2, call an (1 GPU): HEAD after the chunk-floor change -- smoke(), pytest -m gpu (incl. the
# pipeline-variant suites), bench N=1
OUT=gpurun_out/r02an; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu_1gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu_1gpu.log
timeout 600 python bench.py > $OUT/bench_n1.json 2> $OUT/bench_n1.err
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/reference_n1.json 2> $OUT/reference_n1.err
