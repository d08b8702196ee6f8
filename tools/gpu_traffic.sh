#!/bin/bash
# Per-config DRAM traffic of the attention stage (roofline.traffic): one
# `ncu --set full` capture per bench workload, restricted to the sts.attend
# NVTX range of an eager bench run. Reports land in gpurun_out/traffic/;
# `python tools/ncu_traffic.py KEY=REPORT ...` folds them into profiles/ncu_traffic.json.
OUT=${OUT:-gpurun_out/traffic}
mkdir -p $OUT
B="python bench.py --eager --steps 1 --warmup 3 --no-cpu-baseline --no-extras --parity-units 0"
NCU="ncu --set full --clock-control none --import-source on --nvtx --nvtx-include sts.attend/ -c ${NCU_COUNT:-2}"
run() { name=$1; shift; timeout 900 $NCU -o $OUT/$name -f $B "$@" > $OUT/$name.log 2>&1; echo "$name rc=$?" >> $OUT/$name.log; tail -1 $OUT/$name.log; }
for c in ${CFGS:-c2 c2R c3 c4}; do
  case $c in
    c2) run c2 --config c2 ;;
    c2R) run c2R --config c2 --mode R ;;
    c2p16) run c2p16 --config c2 --page-size 16 ;;
    c3) run c3 --config c3 ;;
    c4) run c4 --config c4 ;;
  esac
done
