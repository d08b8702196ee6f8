#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 200 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline"
: > gpurun_out/ab.log
for rep in 1 2; do echo "== run" >> gpurun_out/ab.log; timeout 300 $B >> gpurun_out/ab.log 2>&1; done
