#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_pipeline.py -q -p no:cacheprovider --timeout 120 > gpurun_out/pytest_pipe.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_pipe.log
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline"
: > gpurun_out/draft.log
for cfg in 0 1 2 3 4; do echo "== cfg $cfg" >> gpurun_out/draft.log; STS_DRAFT_CFG=$cfg timeout 200 $B >> gpurun_out/draft.log 2>&1; done
