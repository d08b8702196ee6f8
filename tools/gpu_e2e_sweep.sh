#!/bin/bash
# e2e (attend_host) sweep: host chunk count x attention schedule at c2
OUT=${OUT:-gpurun_out/e2e}
mkdir -p $OUT
for ch in 1 2 3 4 6 8; do for sc in 0 1 3 6; do
STS_HOST_CHUNKS=$ch timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras --parity-units 0 --schedule $sc > $OUT/c${ch}_s${sc}.log 2>&1
python -c "
import json
for l in open('$OUT/c${ch}_s${sc}.log'):
    if l.startswith('{'):
        d=json.loads(l); print('chunks $ch schedule $sc attend', d['value'], 'e2e', d['e2e']['value'])
" || echo "chunks $ch schedule $sc failed"
done; done
