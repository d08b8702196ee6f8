#!/bin/bash
# A/B of library variants, alternating, same box
mkdir -p gpurun_out
B="python bench.py --steps 30 --warmup 5 --no-cpu-baseline"
: > gpurun_out/ab.log
for rep in 1 2 3; do
  echo "== A default" >> gpurun_out/ab.log; timeout 200 $B >> gpurun_out/ab.log 2>&1
  for v in paper_2605_15508_b200/_lib/variants/*.so; do echo "== B $v" >> gpurun_out/ab.log; STS_B200_LIB=$PWD/$v timeout 200 $B >> gpurun_out/ab.log 2>&1; done
done
