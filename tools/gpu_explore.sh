#!/bin/bash
# overhead-vs-bytes sweep, layouts, and ncu source captures of the three gather modes
mkdir -p gpurun_out
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
: > gpurun_out/explore.log
for ctx in 32768 65536 131072; do echo "== ctx $ctx" >> gpurun_out/explore.log; timeout 300 $B --context $ctx >> gpurun_out/explore.log 2>&1; done
echo "== interleaved" >> gpurun_out/explore.log; timeout 300 $B --layout interleaved >> gpurun_out/explore.log 2>&1
echo "== page16" >> gpurun_out/explore.log; timeout 300 $B --page-size 16 >> gpurun_out/explore.log 2>&1
echo "== page16 interleaved" >> gpurun_out/explore.log; timeout 300 $B --page-size 16 --layout interleaved >> gpurun_out/explore.log 2>&1
P="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
# warm-up steps launch: lse, probs, select, decode(sparse), decode(dense) x3 -> capture the 4th step's kernels
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:gather_kernel" -s 12 -c 4 -o gpurun_out/prof_gather $P > gpurun_out/ncu_gather.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_gather.log
tail -2 gpurun_out/ncu_gather.log
