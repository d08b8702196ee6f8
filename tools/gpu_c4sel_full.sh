#!/bin/bash
# c4 select kernels under ncu --set full (one launch each): keys, hist, emit_bits, emit_write
OUT=${OUT:-gpurun_out/c4self}
mkdir -p $OUT
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"dist_keys|dist_hist|dist_emit_bits|dist_emit_write" -c 5 -o $OUT/sel -f python bench.py --config c4 --eager --steps 1 --warmup 0 --no-cpu-baseline --no-extras --parity-units 0 > $OUT/ncu.log 2>&1
for i in 0 1 2 3 4; do python tools/ncu_lines.py $OUT/sel.ncu-rep --launch $i --top 14 --sort stall > $OUT/lines$i.txt 2>&1; done
ncu -i $OUT/sel.ncu-rep --page details --csv > $OUT/details.csv 2>&1
python - <<PY
import csv
rows=list(csv.reader(open("$OUT/details.csv")))
h=rows[0]
for r in rows[1:]:
    d=dict(zip(h,r))
    if d.get("Metric Name") in ("Duration","Achieved Occupancy","Registers Per Thread","DRAM Throughput","Executed Ipc Active","Issue Slots Busy","Block Limit Registers","Block Limit Shared Mem"):
        print(d["ID"], d["Kernel Name"][:40], d["Metric Name"], d["Metric Value"], d["Metric Unit"])
PY
rm -f $OUT/sel.ncu-rep
