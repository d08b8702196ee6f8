#!/bin/bash
# bench variants: token vs page selection, separate vs interleaved K|V layout
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attention.py -q -x -p no:cacheprovider > gpurun_out/pytest_attn.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_attn.log
for v in "--layout separate --page-size 1" "--layout interleaved --page-size 1" "--layout separate --page-size 16" "--layout interleaved --page-size 16"; do
  echo "== $v" >> gpurun_out/variants.log
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline $v >> gpurun_out/variants.log 2>&1
done
