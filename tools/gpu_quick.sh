#!/bin/bash
# tests + bench + ncu of the gather kernels (one timed step)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:gather_kernel" -s 3 -c 4 -o gpurun_out/prof_gather $B > gpurun_out/ncu_gather.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_gather.log
