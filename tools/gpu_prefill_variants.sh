#!/bin/bash
# sparse prefill (and c1) timing: default library vs _lib/variants/*.so
mkdir -p gpurun_out
: > gpurun_out/prefill_variants.log
for so in default paper_2605_15508_b200/_lib/variants/*.so; do
  if [ "$so" = default ]; then E=""; else E="STS_B200_LIB=$so"; fi
  echo "## $(basename $so)" >> gpurun_out/prefill_variants.log
  env $E timeout 300 python tools/bench_prefill.py --n 4096 >> gpurun_out/prefill_variants.log 2>&1
  env $E timeout 300 python tools/bench_prefill.py --n 16384 --iters 3 >> gpurun_out/prefill_variants.log 2>&1
  env $E timeout 300 python bench.py --config c1 --steps 10 --warmup 3 --no-cpu-baseline >> gpurun_out/prefill_variants.log 2>&1
done
