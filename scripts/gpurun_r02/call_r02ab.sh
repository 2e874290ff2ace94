# round 2, call ab (4 GPUs): xall step time vs size at N = 2 and 4 (fixed per-step cost vs streaming rate)
OUT=gpurun_out/r02ab; mkdir -p $OUT
for N in 2 4; do
  T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29545"
  for n in 4000000 8000000 16000000 25557032 51114064 102228128 138357544; do
    timeout 300 $T bench.py --gpus $N --workload xall --size $n --steps 60 --e2e-steps 1 --no-extras 2>$OUT/err.txt | grep '^{' > $OUT/tmp.json
    echo "N=$N n=$n $(python scripts/show_bench.py $OUT/tmp.json)" >> $OUT/size_sweep.txt
  done
done
