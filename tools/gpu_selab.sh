#!/bin/bash
# select kernel A/B: GPU select/pipeline/measured tests, c2 bench with the
# variants in VARS (env assignments), ncu of the
# default select launch (per-line instructions and stalls)
OUT=${OUT:-gpurun_out/selab}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_select.py tests/test_gpu_pipeline.py tests/test_gpu_measured.py -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
for v in ${VARS:-STS_NONE=0}; do
 env $v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras --parity-units 0 ${BENCH} > $OUT/b_$v.log 2>&1
 python -c "
import json
for l in open('$OUT/b_$v.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$v', 'attend', d['value'], 'mask', d.get('mask_build_us'))
" || tail -3 $OUT/b_$v.log
done
if [ -z "$NO_NCU" ]; then
timeout 600 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include sts.select/ -c 1 -o $OUT/sel0 -f python bench.py --eager --steps 1 --warmup 1 --no-cpu-baseline --no-extras --parity-units 0 ${BENCH} > $OUT/ncu0.log 2>&1
ncu -i $OUT/sel0.ncu-rep --page details --csv > $OUT/sel0.details.csv 2>&1
python tools/ncu_lines.py $OUT/sel0.ncu-rep --launch 0 --top 60 --sort inst > $OUT/sel0.lines.txt 2>&1
grep -h '"Duration"\|"Executed Ipc Active"\|"Issue Slots Busy"' $OUT/sel0.details.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
fi
