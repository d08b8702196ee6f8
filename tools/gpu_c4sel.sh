#!/bin/bash
# c4 (1M) select stage: per-kernel durations (ncu launch list of the sts.select NVTX range) + a full
# capture of the keys kernel
OUT=${OUT:-gpurun_out/c4sel}
mkdir -p $OUT
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"dist_" --csv --log-file $OUT/launches.csv python bench.py --config ${CFG:-c4} --eager --steps 1 --warmup 0 --no-cpu-baseline --no-extras --parity-units 0 > $OUT/ncu.log 2>&1
python - <<PY
import csv, collections
rows = list(csv.reader(open("$OUT/launches.csv")))
hdr = None; agg = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID": hdr = r; continue
    if hdr is None or len(r) != len(hdr): continue
    d = dict(zip(hdr, r)); k = d["Kernel Name"][:60]; m = d["Metric Name"]
    try: v = float(d["Metric Value"].replace(",", ""))
    except ValueError: continue
    agg.setdefault(k, collections.defaultdict(float))[m] += v
for k, m in agg.items():
    print(f"{k:60s} {m.get('gpu__time_duration.sum',0)/1e3:9.1f} us  rd {m.get('dram__bytes_read.sum',0)/1e9:6.2f} GB  wr {m.get('dram__bytes_write.sum',0)/1e9:6.2f} GB")
PY
