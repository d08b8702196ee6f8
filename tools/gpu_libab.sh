#!/bin/bash
# A/B of library variants on one box: bench line per library (capture/select/attend timings)
OUT=${OUT:-gpurun_out/libab}
mkdir -p $OUT
for lib in default ${VARIANTS}; do
  if [ "$lib" = default ]; then L=""; else L="STS_B200_LIB=paper_2605_15508_b200/_lib/variants/libsts_b200_$lib.so"; fi
  env $L timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras --parity-units 0 ${BENCH} > $OUT/$lib.log 2>&1
  python -c "
import json,sys
for l in open('$OUT/$lib.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$lib', 'attend', d['value'], d.get('mask_build_us'))
" || tail -3 $OUT/$lib.log
done
