#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/sweep.log
for cfg in 0 1 2 3; do
  for ps in 1; do
    echo "== cfg $cfg ps $ps" >> gpurun_out/sweep.log
    STS_GATHER_CFG=$cfg timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --page-size $ps >> gpurun_out/sweep.log 2>&1
  done
done
