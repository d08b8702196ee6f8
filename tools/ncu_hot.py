#!/usr/bin/env python
"""Summarise an ncu report's source page: CUDA lines ranked by warp-stall
samples and executed instructions (needs -lineinfo builds).

    python tools/ncu_hot.py gpurun_out/prof.ncu-rep [--top 25] [--kernel regex]
"""

import argparse
import csv
import io
import re
import subprocess
import sys


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--top", type=int, default=25)
    ap.add_argument("--launch", type=int, default=None, help="--print-details launch index filter (ncu -l)")
    a = ap.parse_args()
    cmd = ["ncu", "-i", a.report, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if a.launch is not None:
        cmd += ["--launch-skip", str(a.launch), "--launch-count", "1"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    agg = {}
    cur_file = "?"
    header = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            header = r
            continue
        if header is None or not r[0].isdigit():
            continue
        d = dict(zip(header, r))
        try:
            samples = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
            inst = int(d.get("Instructions Executed", "0") or 0)
        except ValueError:
            continue
        key = (cur_file, int(r[0]))
        s0, i0, src = agg.get(key, (0, 0, r[1]))
        agg[key] = (s0 + samples, i0 + inst, src)
    tot_s = sum(v[0] for v in agg.values()) or 1
    tot_i = sum(v[1] for v in agg.values()) or 1
    print(f"total stall samples {tot_s}, instructions {tot_i}")
    for (f, ln), (s, i, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[: a.top]:
        print(f"{100 * s / tot_s:5.1f}% samp {100 * i / tot_i:5.1f}% inst  {f}:{ln:<4} {src.strip()[:90]}")


if __name__ == "__main__":
    main()
