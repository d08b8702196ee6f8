#!/usr/bin/env python
"""Per-source-line warp-instruction counts of one launch in an ncu report."""
import csv, io, subprocess, sys
rep, launch = sys.argv[1], sys.argv[2]
units = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--launch-skip", launch, "--launch-count", "1"], capture_output=True, text=True).stdout
agg, header, cur = {}, None, "?"
def toint(x):
    try: return int(x)
    except ValueError: return 0
for r in csv.reader(io.StringIO(out)):
    if not r: continue
    if r[0] == "File Path": cur = r[1].split('/')[-1]; continue
    if r[0] == "Line No": header = r; continue
    if header is None or not r[0].isdigit(): continue
    d = dict(zip(header, r))
    i = toint(d.get("Instructions Executed", "0")); smp = toint(d.get("Warp Stall Sampling (All Samples)", "0"))
    key = (cur, int(r[0])); a = agg.get(key, (0, 0, r[1])); agg[key] = (a[0] + i, a[1] + smp, r[1])
tot = sum(v[0] for v in agg.values()); tots = sum(v[1] for v in agg.values()) or 1
print(f"total warp-instructions {tot}  per unit {tot/units:.1f}")
for (f, ln), (i, smp, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*i/tot:5.1f}% inst {i/units:7.1f}/u {100*smp/tots:5.1f}% stall {f}:{ln} {src.strip()[:70]}")
