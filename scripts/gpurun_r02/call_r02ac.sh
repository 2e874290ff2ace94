# round 2, call ac (4 GPUs): per-iteration timeline (SIG times, producer flag waits) of the cross kernel
OUT=${OUT:-gpurun_out/r02ac}; mkdir -p $OUT
for N in 2 4; do
  T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29545"
  [ -n "$NOPERF" ] || timeout 300 $T bench.py --gpus $N --workload xall --steps 60 --e2e-steps 1 --no-extras 2>$OUT/err.txt | grep '^{' > $OUT/tmp.json
  echo "N=$N xall (no profiling) $(python scripts/show_bench.py $OUT/tmp.json)" >> $OUT/perf.txt
  for spec in "xall:0" "xall:4000000" "cfg3:0"; do
    wl=${spec%%:*}; sz=${spec##*:}
    tag=tl_${wl}_${sz}_n$N
    RP_XGPU_PROFILE=$OUT/$tag timeout 300 $T bench.py --gpus $N --workload $wl --size $sz --steps 20 --no-e2e --no-extras > $OUT/$tag.json 2>&1
    files=""; for r in $(seq 0 $((N-1))); do files="$files $OUT/$tag.$r"; done
    python scripts/xgpu_timeline.py $files > $OUT/timeline_$tag.txt 2>&1
  done
done
