#!/bin/bash
# Round-2 evidence run on one B200: GPU suite, smoke, default bench (+ CPU
# baseline, mode-R / fp32 side lines), reference arm, c4 one-GPU, c3 sparsity
# sweep, per-config attention traffic (ncu), launch list, ncu --set full of the
# step's kernels, offload / block-sparse prefill / generate benches, gather probe.
O=${O:-gpurun_out/r2final}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.log 2>&1; echo "ref rc=$?" >> $O/bench_ref.log
timeout 900 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c4.log 2>&1; echo "c4 rc=$?" >> $O/bench_c4.log
: > $O/bench_c3.log
for sp in 0.5 0.75 0.9 0.95 0.98; do timeout 600 python bench.py --config c3 --sparsity $sp --steps 5 --warmup 3 --no-cpu-baseline --no-extras >> $O/bench_c3.log 2>&1; done
echo "c3 rc=$?" >> $O/bench_c3.log
timeout 900 python tools/bench_offload.py 32 16 > $O/offload.log 2>&1
timeout 900 python tools/bench_prefill_tc.py > $O/prefill_tc.log 2>&1
timeout 600 python tools/bench_generate.py > $O/generate.log 2>&1
python tools/gather_probe.py --build > /dev/null 2>&1 && timeout 300 python tools/gather_probe.py > $O/gather_probe.json 2>&1
P="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras --eager --parity-units 0"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $P > $O/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:verify_decode|merge_pieces|select_kernel|select_reg_kernel|capture_kernel" -s 10 -c 6 -o $O/prof_step -f $P > $O/ncu_step.log 2>&1
python tools/ncu_summary.py $O/prof_step.ncu-rep --json $O/ncu_step_summary.json > /dev/null 2>&1
python tools/ncu_hot.py $O/prof_step.ncu-rep --top 40 > $O/ncu_step_hot.txt 2>&1
rm -f $O/prof_step.ncu-rep
OUT=$O/traffic CFGS="c2 c2R c3 c4" bash tools/gpu_traffic.sh
python tools/ncu_traffic.py --out=$O/ncu_traffic.json "c2:S:s0.9:ps1:separate:P1=$O/traffic/c2.ncu-rep" "c2:R:s0.9:ps1:separate:P1=$O/traffic/c2R.ncu-rep" "c3:S:s0.9:ps1:separate:P1=$O/traffic/c3.ncu-rep" "c4:S:s0.9:ps1:separate:P1=$O/traffic/c4.ncu-rep" > $O/traffic.log 2>&1
rm -f $O/traffic/*.ncu-rep
du -sh $O
for f in $O/pytest_gpu.log $O/smoke.log $O/bench.log $O/bench_ref.log $O/bench_c4.log; do tail -n 2 $f | cut -c1-300; done
