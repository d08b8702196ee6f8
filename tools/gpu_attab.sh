#!/bin/bash
# attention iteration: attention/pipeline/measured GPU tests, c2 bench line,
# per-CTA timeline (STS_TRACE variant) and the gather probe
OUT=${OUT:-gpurun_out/attab}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_pipeline.py tests/test_gpu_measured.py -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log
for i in 1 2; do
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras --parity-units 0 ${BENCH} > $OUT/bench$i.log 2>&1
python -c "
import json
for l in open('$OUT/bench$i.log'):
    if l.startswith('{'):
        d=json.loads(l); print('attend', d['value'], 'frac', d['roofline']['frac'], 'mask', d.get('mask_build_us'), 'e2e', d['e2e']['value'])
" || tail -3 $OUT/bench$i.log
done
if [ -f paper_2605_15508_b200/_lib/variants/libsts_b200_trace.so ]; then
STS_B200_LIB=paper_2605_15508_b200/_lib/variants/libsts_b200_trace.so timeout 300 python tools/trace_decode.py > $OUT/trace.json 2>&1
python -c "
import json; d=json.load(open('$OUT/trace.json'))['sparse']
print({k: d[k] for k in ('first_tile','loop_end','exit')})"
fi
[ -f tools/_build/gather_probe.so ] && timeout 300 python tools/gather_probe.py > $OUT/gather.json 2>&1 && cat $OUT/gather.json
