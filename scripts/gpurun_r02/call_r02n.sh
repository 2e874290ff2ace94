# round 2, call n (1 GPU): ncu evidence -- launch list of the default bench (N=1), full capture of the
# intra-GPU kernel at configs[1] and of the warp-specialized cross kernel (2 emulated GPUs, R50 size)
OUT=gpurun_out/r02n; mkdir -p $OUT
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1"
E="python scripts/emul_case.py 2 1 25557032"
$B > $OUT/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_default_n1.csv $B > $OUT/ncu_launches.log 2>&1
$B > $OUT/plain_bench2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:preduce_dyn -s 4 -c 1 -o $OUT/prof_dyn $B > $OUT/ncu_dyn.log 2>&1
$E > $OUT/plain_emul.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:xgpu_ws_emul -s 1 -c 1 -o $OUT/prof_ws_emul $E > $OUT/ncu_ws.log 2>&1
ls -la $OUT
