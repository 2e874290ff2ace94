# round 2, call aj (1 GPU): ncu --set full of the warp-specialized cross kernel at HEAD
# (2 emulated GPUs, ResNet-50 size; dynamic claiming, two-SIG pipeline with early A flags)
OUT=gpurun_out/r02aj; mkdir -p $OUT
E="python scripts/emul_case.py 2 1 25557032"
$E > $OUT/plain_emul.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:xgpu_ws_emul -s 1 -c 1 -o $OUT/prof_ws_emul $E > $OUT/ncu_ws.log 2>&1
ls -la $OUT
