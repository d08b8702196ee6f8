#!/bin/bash
# bench the default library against _lib/variants/*.so on c2 and c3 (one line each)
mkdir -p gpurun_out
: > gpurun_out/variant_bench.log
for cfg in ${CFGS:-c2 c3}; do
  echo "## $cfg default" >> gpurun_out/variant_bench.log
  timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline >> gpurun_out/variant_bench.log 2>&1
  for so in paper_2605_15508_b200/_lib/variants/*.so; do
    echo "## $cfg $(basename $so)" >> gpurun_out/variant_bench.log
    STS_B200_LIB=$so timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline >> gpurun_out/variant_bench.log 2>&1
  done
done
grep -c '^{' gpurun_out/variant_bench.log
