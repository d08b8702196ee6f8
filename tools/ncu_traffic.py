#!/usr/bin/env python
"""Per-config DRAM traffic of the attention stage, for bench.py's
``roofline.traffic``.

Reads ``ncu --set full`` reports of ``bench.py --eager`` restricted to the
``sts.attend`` NVTX range (tools/gpu_traffic.sh) and writes
profiles/ncu_traffic.json: {workload_key: {"dram_bytes": read+write bytes of
the attention stage per launch (main kernel + piece merge, if any),
"kernels": [...], "source": report name}}.

    python tools/ncu_traffic.py KEY=gpurun_out/traffic/c2.ncu-rep [KEY=...]
"""

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "tools"))
from ncu_summary import summarize  # noqa: E402


def main(argv):
    out = ROOT / "profiles" / "ncu_traffic.json"
    if argv and argv[0].startswith("--out="):
        out = Path(argv[0].split("=", 1)[1])
        argv = argv[1:]
    db = json.loads(out.read_text()) if out.exists() else {}
    for arg in argv:
        key, rep = arg.split("=", 1)
        rows = summarize(rep)
        if not rows:
            print(f"{key}: no kernels in {rep}")
            continue
        # one attention stage = the launches of one replay of sts.attend; the
        # report holds a whole number of stages (-c), average per stage
        names = [r["kernel"] for r in rows]
        main_idx = [i for i, n in enumerate(names) if "verify_decode_kernel" in n]
        stages = max(1, len(main_idx))
        dram = sum((r["dram_read_MB"] or 0) + (r["dram_write_MB"] or 0) for r in rows) * 1e6 / stages
        dur = sum(r["dur_us"] or 0 for r in rows) / stages
        db[key] = {"dram_bytes": int(round(dram)), "ncu_us_per_stage": round(dur, 2),
                   "kernels": sorted(set(n[:80] for n in names)), "launches_per_stage": len(rows) / stages,
                   "source": f"ncu --set full of bench.py --eager, NVTX range sts.attend ({Path(rep).name})"}
        print(key, db[key])
    out.write_text(json.dumps(db, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main(sys.argv[1:])
