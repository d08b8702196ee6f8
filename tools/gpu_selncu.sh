#!/bin/bash
# ncu --set full of the select stage (c2) for the default library and STS_SELECT_SMEM=1
OUT=${OUT:-gpurun_out/selncu}
mkdir -p $OUT
for v in 0 1; do
  STS_SELECT_SMEM=$v timeout 600 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include sts.select/ -c 1 -o $OUT/sel$v -f python bench.py --eager --steps 1 --warmup 1 --no-cpu-baseline --no-extras --parity-units 0 > $OUT/ncu$v.log 2>&1
  ncu -i $OUT/sel$v.ncu-rep --page details --csv > $OUT/sel$v.details.csv 2>&1
  python tools/ncu_lines.py $OUT/sel$v.ncu-rep --launch 0 --top 60 --sort stall > $OUT/sel$v.lines.txt 2>&1
done
grep -h "Duration\|Registers\|Achieved Occupancy\|Issue Slots Busy\|DRAM Throughput\|Executed Ipc A" $OUT/sel*.details.csv | cut -c1-200
