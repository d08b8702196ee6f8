#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 120 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/bench_prefill.py --n 4096 > gpurun_out/prefill.log 2>&1
timeout 300 python tools/bench_prefill.py --n 16384 --iters 3 >> gpurun_out/prefill.log 2>&1
