#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 90 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
: > gpurun_out/dyn.log
for f in 0 0.1 0.2 0.3; do for c in 2 4 8; do echo "== frac $f chunk $c" >> gpurun_out/dyn.log; STS_DYN_FRAC=$f STS_DYN_CHUNK=$c timeout 120 $B >> gpurun_out/dyn.log 2>&1; done; done
echo "== legacy" >> gpurun_out/dyn.log; STS_DECODE_LEGACY=1 timeout 120 $B >> gpurun_out/dyn.log 2>&1
STS_B200_LIB=$PWD/paper_2605_15508_b200/_lib/variants/libsts_b200_trace.so timeout 120 python tools/trace_decode.py 32768 > gpurun_out/trace_32k.json 2>&1
