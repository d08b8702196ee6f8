#!/bin/bash
# Round-2 call A: GPU suite, default bench line, per-config attention traffic (ncu).
mkdir -p gpurun_out/r2a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2a/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2a/pytest.log
timeout 600 python bench.py > gpurun_out/r2a/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/r2a/bench.log
bash tools/gpu_traffic.sh
tail -3 gpurun_out/r2a/pytest.log; tail -2 gpurun_out/r2a/bench.log
