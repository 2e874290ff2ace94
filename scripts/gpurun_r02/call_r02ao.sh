# round 2, call ao (4 GPUs): the full multi-GPU suite at HEAD (after the chunk-floor change)
OUT=gpurun_out/r02ao; mkdir -p $OUT
timeout 1100 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider > $OUT/pytest_multi_4gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_multi_4gpu.log
