#!/bin/bash
# bench variants: mode R, page mode, interleaved KV layout, c1 (each one line)
mkdir -p gpurun_out
: > gpurun_out/variants.log
for args in "--mode R" "--page-size 16" "--mode R --page-size 16" "--layout interleaved" "--config c1" "--config c3 --mode R"; do
  echo "## $args" >> gpurun_out/variants.log
  timeout 600 python bench.py $args --steps 5 --warmup 3 --no-cpu-baseline >> gpurun_out/variants.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_R.csv python bench.py --mode R --steps 1 --warmup 3 --no-cpu-baseline --eager > /dev/null 2>&1
grep -c '^{' gpurun_out/variants.log
