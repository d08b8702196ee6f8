#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 90 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
mkdir -p gpurun_out
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
: > gpurun_out/iter.log
echo "== default" >> gpurun_out/iter.log; timeout 200 $B >> gpurun_out/iter.log 2>&1
P="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --eager"
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:verify_decode|merge_pieces" -s 18 -c 6 -o gpurun_out/prof_gather $P > gpurun_out/ncu_gather.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_gather.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $P > /dev/null 2>&1
