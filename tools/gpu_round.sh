#!/bin/bash
# Full evidence run: GPU tests, smoke, default bench (+CPU baseline), reference arm,
# c4 (1M) single-GPU, c3 sparsity sweep, launch list + ncu --set full of the hot kernels.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 120 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; echo "c4 rc=$?" >> gpurun_out/bench_c4.log
: > gpurun_out/bench_c3.log
for sp in 0.5 0.75 0.9 0.95 0.98; do timeout 600 python bench.py --config c3 --sparsity $sp --steps 5 --warmup 3 --no-cpu-baseline >> gpurun_out/bench_c3.log 2>&1; done
echo "c3 rc=$?" >> gpurun_out/bench_c3.log
P="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --eager"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $P > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:verify_decode|merge_pieces|select_kernel" -s 30 -c 6 -o gpurun_out/prof_step $P > gpurun_out/ncu_step.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_step.log
for f in gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/bench.log gpurun_out/bench_ref.log gpurun_out/bench_c4.log; do tail -n 2 $f; done
