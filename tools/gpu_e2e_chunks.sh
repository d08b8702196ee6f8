#!/bin/bash
# e2e (attend_host) vs STS_HOST_CHUNKS
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_pipeline.py -q -x -p no:cacheprovider -k host_buffer > gpurun_out/pt.log 2>&1; tail -1 gpurun_out/pt.log
: > gpurun_out/e2e_chunks.log
for D in 0 1; do for c in 1 2 3; do
  echo "## chunks=$c direct=$D" >> gpurun_out/e2e_chunks.log
  STS_HOST_DIRECT=$D STS_HOST_CHUNKS=$c timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline >> gpurun_out/e2e_chunks.log 2>&1
done; done
