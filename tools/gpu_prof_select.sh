#!/bin/bash
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:select_kernel" -s 1 -c 1 -o gpurun_out/prof_select $B > gpurun_out/ncu_select.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_select.log
