"""Summarise gpurun_out/variant_bench.log (or a given file): value, capture, select, step."""
import json
import sys

cur = None
for line in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/variant_bench.log"):
    if line.startswith("##"):
        cur = line[2:].strip()
    elif line.startswith("{"):
        d = json.loads(line)
        mb = d.get("mask_build_us", {})
        print(f"{cur:40s} attend {d['value']:9.2f}  capture {mb.get('draft_capture', 0):9.2f}  "
              f"select {mb.get('select', 0):9.2f}  step {d.get('sts_step_us', 0):9.2f}  frac {d['roofline']['frac']}")
