OUT=gpurun_out/ts; mkdir -p $OUT
timeout 600 ncu --set full --import-source on --clock-control none -k regex:select_kernel -c 1 -o $OUT/ts -f python tools/bench_prefill_tc.py --n 16384 --iters 1 > $OUT/ncu.log 2>&1
python tools/ncu_lines.py $OUT/ts.ncu-rep --launch 0 --top 40 --sort stall > $OUT/ts.lines.txt 2>&1
ncu -i $OUT/ts.ncu-rep --page details --csv > $OUT/ts.details.csv 2>&1
grep -h '"Duration"\|"Executed Ipc Active"\|"Issue Slots Busy"\|"Registers Per Thread"' $OUT/ts.details.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
