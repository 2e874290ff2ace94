# round 2, call z (4 GPUs): poisoned-staging race check (emulated + 2/4 GPUs), watchdog, momentum, native
OUT=gpurun_out/r02z; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_emulated.py -m gpu -q -p no:cacheprovider > $OUT/pytest_emul.log 2>&1; echo "rc=$?" >> $OUT/pytest_emul.log
timeout 1500 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider -k "poison or watchdog or momentum or native" > $OUT/pytest_multi.log 2>&1; echo "rc=$?" >> $OUT/pytest_multi.log
