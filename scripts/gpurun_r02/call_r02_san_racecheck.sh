# round 2 (1 GPU): compute-sanitizer --tool racecheck on the hot kernels (intra-GPU dynamic-tile kernel, forced at a
# small size; warp-specialized cross kernel on 2 and 3 emulated GPUs), one tool per call
OUT=gpurun_out/r02_san; mkdir -p $OUT
RP_DYN_MIN_BYTES=0 timeout 600 python scripts/sanitize_case.py > $OUT/plain_racecheck.log 2>&1 && \
RP_DYN_MIN_BYTES=0 timeout 1500 compute-sanitizer --tool racecheck --print-limit 50 python scripts/sanitize_case.py > $OUT/racecheck.log 2>&1
echo "rc=$?" >> $OUT/racecheck.log
