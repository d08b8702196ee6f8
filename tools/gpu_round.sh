#!/bin/bash
# One gpurun call: GPU tests, smoke, bench (+reference arm), gather-config sweep,
# launch list and ncu --set full captures of the two hot kernels.  Logs -> gpurun_out/
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
: > gpurun_out/sweep.log
for cfg in 0 1 2 3; do
  echo "== cfg $cfg" >> gpurun_out/sweep.log
  STS_GATHER_CFG=$cfg timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline >> gpurun_out/sweep.log 2>&1
done
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?" >> gpurun_out/ncu_launches.log
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:gather_kernel" -s 0 -c 6 -o gpurun_out/prof_gather $B > gpurun_out/ncu_gather.log 2>&1
echo "gather rc=$?" >> gpurun_out/ncu_gather.log
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:select_kernel" -s 3 -c 1 -o gpurun_out/prof_select $B > gpurun_out/ncu_select.log 2>&1
echo "select rc=$?" >> gpurun_out/ncu_select.log
for f in gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/bench.log gpurun_out/bench_ref.log; do tail -n 3 $f; done
