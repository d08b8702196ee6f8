#!/bin/bash
# pipeline-shape sweep of the verify decode kernel (STS_VERIFY_CFG) x KV layout / page size
mkdir -p gpurun_out
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
: > gpurun_out/sweep.log
for cfg in 0 1 2 3 4; do
  for v in "" "--layout interleaved" "--page-size 16 --layout interleaved"; do
    echo "== cfg $cfg $v" >> gpurun_out/sweep.log
    STS_VERIFY_CFG=$cfg timeout 300 $B $v >> gpurun_out/sweep.log 2>&1
  done
done
echo "== legacy" >> gpurun_out/sweep.log; STS_DECODE_LEGACY=1 timeout 300 $B >> gpurun_out/sweep.log 2>&1
echo "== legacy interleaved" >> gpurun_out/sweep.log; STS_DECODE_LEGACY=1 timeout 300 $B --layout interleaved >> gpurun_out/sweep.log 2>&1
