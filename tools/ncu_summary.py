#!/usr/bin/env python
"""Per-launch headline metrics of an ncu report (raw page), one line per kernel.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--json out.json]
"""

import argparse
import csv
import io
import json
import subprocess

METRICS = {
    "dur_us": ("gpu__time_duration.sum", 1),
    "dram_read_MB": ("dram__bytes_read.sum", 1e-6),
    "dram_write_MB": ("dram__bytes_write.sum", 1e-6),
    "dram_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "sm_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", 1),
    "ipc": ("sm__inst_executed.avg.per_cycle_active", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "regs": ("launch__registers_per_thread", 1),
    "tensor_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1),
}


def to_float(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


def summarize(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(head, r))
        u = dict(zip(head, units))
        item = {"kernel": d.get("Kernel Name", "")[:90]}
        for k, (m, scale) in METRICS.items():
            v = to_float(d.get(m))
            unit = u.get(m, "")
            if v is not None and m.startswith("dram__bytes"):
                mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
                v = v * mult * scale
            elif v is not None and m == "gpu__time_duration.sum":
                # -> microseconds
                mult = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}.get(unit, 1)
                v = v * mult * scale
            item[k] = None if v is None else round(v, 2)
        res.append(item)
    return res


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--json")
    a = ap.parse_args()
    res = summarize(a.report)
    for it in res:
        print(json.dumps(it))
    if a.json:
        open(a.json, "w").write(json.dumps(res, indent=1))
