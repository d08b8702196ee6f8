#!/bin/bash
# prefill iteration: tcgen05 prefill parity tests, bench_prefill_tc, ncu of the dense 16K launch
OUT=${OUT:-gpurun_out/pf}
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_prefill_tc.py -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log
timeout 600 python tools/bench_prefill_tc.py ${PFN:---n 4096 16384 32768} > $OUT/bench.log 2>&1
python -c "
import json
for l in open('$OUT/bench.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['workload'][60:80], 'sel', d['tile_select_us'], 'selg', d.get('tile_select_graph_us'), 'sparse', d['sparse_prefill_us'], 'dense', d['dense_same_kernel_us'], 'TF/s', d['dense_same_kernel_TFLOPs'], 'fa', d['dense_flash_attn_us'])
" || tail -3 $OUT/bench.log
if [ -z "$NO_NCU" ]; then
timeout 600 ncu --set full --import-source on --clock-control none -k regex:prefill_tc -s 4 -c 1 -o $OUT/pf -f python tools/bench_prefill_tc.py --n 16384 --iters 1 > $OUT/ncu.log 2>&1
ncu -i $OUT/pf.ncu-rep --page details --csv > $OUT/pf.details.csv 2>&1
python tools/ncu_lines.py $OUT/pf.ncu-rep --launch 0 --top 50 --sort stall > $OUT/pf.lines.txt 2>&1
grep -h '"Duration"\|"Executed Ipc Active"\|"Issue Slots Busy"' $OUT/pf.details.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
fi
