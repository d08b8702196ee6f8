#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 200 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline"
: > gpurun_out/ab.log
echo "== cluster select" >> gpurun_out/ab.log; timeout 300 $B > gpurun_out/bench.log 2>&1; cat gpurun_out/bench.log >> gpurun_out/ab.log
echo "== single-cta select" >> gpurun_out/ab.log; STS_SELECT_CLUSTER=0 timeout 300 $B >> gpurun_out/ab.log 2>&1
