#!/usr/bin/env python
"""Per-source-line instruction counts and stall samples of one launch in an ncu report.

    python tools/ncu_lines.py report.ncu-rep --launch 2 [--top 40] [--sort inst|stall]
"""
import argparse, csv, io, subprocess

ap = argparse.ArgumentParser()
ap.add_argument("report")
ap.add_argument("--launch", type=int, default=0)
ap.add_argument("--top", type=int, default=40)
ap.add_argument("--sort", default="inst")
a = ap.parse_args()
out = subprocess.run(["ncu", "-i", a.report, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--launch-skip", str(a.launch), "--launch-count", "1"], capture_output=True, text=True).stdout
agg, cur, header = {}, "?", None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        header = r
        continue
    if header is None or not r[0].isdigit():
        continue
    d = dict(zip(header, r))
    try:
        inst = int(d.get("Instructions Executed", "0") or 0)
        st = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        continue
    k = (cur, int(r[0]))
    i0, s0, src = agg.get(k, (0, 0, r[1]))
    agg[k] = (i0 + inst, s0 + st, src)
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"instructions {ti}  stall samples {ts}")
key = (lambda kv: -kv[1][0]) if a.sort == "inst" else (lambda kv: -kv[1][1])
acc = 0
for (f, ln), (i, s, src) in sorted(agg.items(), key=key)[: a.top]:
    acc += i
    print(f"{100*i/ti:5.1f}% inst ({100*acc/ti:5.1f} cum) {100*s/ts:5.1f}% stall  {f}:{ln:<4} {src.strip()[:80]}")
