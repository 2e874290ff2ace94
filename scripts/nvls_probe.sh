#!/bin/bash
OUT=gpurun_out/$1; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/nvls_probe scripts/nvls_probe.cu -lcuda > $OUT/build.log 2>&1
for KP in 2 3 4; do
  for U in 1 2 4 8; do
    for C in 1 2; do
      timeout 60 /tmp/nvls_probe $KP 25557032 $C 256 $U | grep -v "^dev\|^granul" >> $OUT/nvls.txt 2>&1
    done
  done
done
timeout 60 /tmp/nvls_probe 4 25557032 1 256 4 1 | grep -v "^dev" >> $OUT/nvls.txt 2>&1
timeout 60 /tmp/nvls_probe 2 134217728 1 256 4 >> $OUT/nvls.txt 2>&1
timeout 60 /tmp/nvls_probe 4 134217728 1 256 4 >> $OUT/nvls.txt 2>&1
