#!/bin/bash
# Sweep the cross-GPU kernel knobs on N GPUs: bash scripts/xgpu_sweep.sh TAG N
TAG=${1:-s01}; N=${2:-2}
OUT=gpurun_out/$TAG; mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533"
for WL in cfg3 cfg4; do
 for U in 1 2 4; do
  for CH in 2048 8192 32768; do
   for CPS in 0 1; do
    RP_XGPU_U=$U RP_XGPU_CHUNK_F4=$CH RP_XGPU_CTAS_PER_SM=$CPS timeout 200 $TR bench.py --gpus $N --steps 30 --warmup 3 --workload $WL --e2e-steps 1 2>/dev/null | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$WL U=$U CH=$CH CPS=$CPS', d['value'], d['ms_per_step'], r['achieved'], r['frac'])" >> $OUT/sweep.txt
   done
  done
 done
done
echo done >> $OUT/sweep.txt
