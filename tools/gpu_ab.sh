#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 120 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
B="python bench.py --steps 30 --warmup 5 --no-cpu-baseline"
: > gpurun_out/ab.log
for rep in 1; do
  echo "== cluster" >> gpurun_out/ab.log; timeout 200 $B >> gpurun_out/ab.log 2>&1
  echo "== streamk" >> gpurun_out/ab.log; STS_VERIFY_CLUSTER=0 timeout 200 $B >> gpurun_out/ab.log 2>&1
done
echo "== cluster c4" >> gpurun_out/ab.log; timeout 300 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline >> gpurun_out/ab.log 2>&1
echo "== streamk c4" >> gpurun_out/ab.log; STS_VERIFY_CLUSTER=0 timeout 300 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline >> gpurun_out/ab.log 2>&1
