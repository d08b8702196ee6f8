#!/bin/bash
# Launch list + one `ncu --set full` capture per hot kernel (1 GPU, short bench).
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?" >> gpurun_out/ncu_launches.log
# decode kernel: launches alternate sparse, dense (warmup step, then timed step)
# per step: draft lse, draft probs, sparse decode, dense decode -> skip the warm-up step's 4
timeout 900 ncu --set full --clock-control none --import-source on \
  -k "regex:sparse_decode_bf16" -s 4 -c 4 -o gpurun_out/prof_decode $B > gpurun_out/ncu_decode.log 2>&1
echo "decode rc=$?" >> gpurun_out/ncu_decode.log
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:select_kernel" -s 1 -c 1 -o gpurun_out/prof_select $B > gpurun_out/ncu_select.log 2>&1
echo "select rc=$?" >> gpurun_out/ncu_select.log
