#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline"
: > gpurun_out/ab.log
echo "== v2" >> gpurun_out/ab.log; timeout 300 $B >> gpurun_out/ab.log 2>&1
echo "== v1" >> gpurun_out/ab.log; STS_SELECT_V2=0 timeout 300 $B >> gpurun_out/ab.log 2>&1
echo "== v2 tie-free? page16" >> gpurun_out/ab.log; timeout 300 $B --page-size 16 >> gpurun_out/ab.log 2>&1
