#!/bin/bash
# c3 launch list + ncu --set full of the capture kernels (LSE, probabilities)
mkdir -p gpurun_out
P="python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline --eager"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv $P > gpurun_out/ncu_c3_launch.log 2>&1; echo "launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:verify_decode" -s 12 -c 2 -o gpurun_out/prof_c3cap $P > gpurun_out/ncu_c3cap.log 2>&1; echo "ncu rc=$?"
