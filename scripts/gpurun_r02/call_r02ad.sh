# round 2, call ad (4 GPUs): host enqueue time vs device time (is the N = 4 start skew host-made?)
OUT=gpurun_out/r02ad; mkdir -p $OUT
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29545"
for wl in xall cfg3; do
  timeout 300 $T bench.py --gpus 4 --workload $wl --steps 60 --e2e-steps 1 --no-extras 2>$OUT/err_$wl.txt | grep '^{' > $OUT/$wl.json
  python -c "import json,sys; d=json.load(open('$OUT/$wl.json')); print('$wl', d['ms_per_step'], d['host_enqueue_ms'], d['steps'])" >> $OUT/host.txt
done
nproc >> $OUT/host.txt
