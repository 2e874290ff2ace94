#!/bin/bash
OUT=gpurun_out/$1; mkdir -p $OUT
for MB in 0 2; do RP_PREDUCE_MINB=$MB python bench.py --steps 200 --warmup 5 --no-cpu-baseline --e2e-steps 1 2>/dev/null | grep '^{' > $OUT/t.json; echo "cfg2 MINB=$MB $(python scripts/show_bench.py $OUT/t.json)" >> $OUT/sweep.txt; done
for MB in 0 3 4; do RP_PREDUCE_MINB=$MB python bench.py --steps 200 --warmup 5 --no-cpu-baseline --e2e-steps 1 --workload cfg2ii 2>/dev/null | grep '^{' > $OUT/t.json; echo "cfg2ii MINB=$MB $(python scripts/show_bench.py $OUT/t.json)" >> $OUT/sweep.txt; done
for MB in 0 2; do RP_PREDUCE_MINB=$MB python bench.py --steps 200 --warmup 5 --no-cpu-baseline --e2e-steps 1 2>/dev/null | grep '^{' > $OUT/t.json; echo "cfg2 MINB=$MB (repeat) $(python scripts/show_bench.py $OUT/t.json)" >> $OUT/sweep.txt; done
