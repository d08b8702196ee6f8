#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
: > gpurun_out/iter.log
for ctx in 32768; do echo "== ctx $ctx" >> gpurun_out/iter.log; timeout 300 $B --context $ctx >> gpurun_out/iter.log 2>&1; done
echo "== legacy" >> gpurun_out/iter.log; STS_DECODE_LEGACY=1 timeout 300 $B >> gpurun_out/iter.log 2>&1
P="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --eager"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:verify_decode|gather_kernel" -s 12 -c 4 -o gpurun_out/prof_gather $P > gpurun_out/ncu_gather.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_gather.log
tail -2 gpurun_out/pytest_gpu.log
