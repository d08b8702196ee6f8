#!/bin/bash
# sharded-path GPU tests + c4 (1M context) bench + its kernel launch list
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_select.py -x -q -p no:cacheprovider --timeout 200 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; echo "bench c4 rc=$?" >> gpurun_out/bench_c4.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --eager > gpurun_out/ncu_c4.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_c4.log
for f in gpurun_out/pytest_gpu.log gpurun_out/bench_c4.log gpurun_out/ncu_c4.log; do tail -n 3 $f | cut -c1-300; done
