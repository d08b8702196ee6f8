#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_attention.py -q -p no:cacheprovider --timeout 200 -k "offload or golden" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python tools/bench_offload.py 8 > gpurun_out/offload.log 2>&1
