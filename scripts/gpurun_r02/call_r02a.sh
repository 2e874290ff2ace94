set -x
OUT=gpurun_out/r02a; mkdir -p $OUT
nvidia-smi topo -m > $OUT/topo.txt 2>&1
python scripts/nvml_nvlink_probe.py > $OUT/nvml_probe.txt 2>&1
bash scripts/gpu_multi.sh r02a 2 "cfg4 cfg3 r50x8"
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29542"
RP_XGPU_PROFILE=$OUT/tl_cfg4 timeout 300 $T bench.py --gpus 2 --workload cfg4 --steps 20 --e2e-steps 1 > $OUT/tl_cfg4.json 2>&1
RP_XGPU_PROFILE=$OUT/tl_r50x8 timeout 300 $T bench.py --gpus 2 --workload r50x8 --steps 20 --e2e-steps 1 > $OUT/tl_r50x8.json 2>&1
python scripts/xgpu_timeline.py $OUT/tl_cfg4.0 $OUT/tl_cfg4.1 $OUT/tl_r50x8.0 $OUT/tl_r50x8.1 > $OUT/timelines.txt 2>&1
