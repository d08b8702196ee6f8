#!/usr/bin/env python
"""Golden vectors for the resident page pool (offload tier, "prefetch"
strategy): random per-step page traces of one (layer, head) unit with
overlapping selections, run through the reference simulator itself
(specsparse.offloadsim.simulate, src/offloadsim.py:173-209) with a one-layer
config whose page transfer time is 1, so each step's `transfer` is its number
of missing pages.  Writes tests/golden/offload_lru.json.

    python tests/golden/make_offload_golden.py   (needs /root/reference)
"""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from specsparse.offloadsim import OffloadConfig, simulate  # noqa: E402

rng = np.random.default_rng(2605)
cases = []
for n_pages, per_step, capacity, steps, churn in ((200, 20, 20, 8, 0.3), (200, 20, 35, 10, 0.5),
                                                  (64, 16, 16, 6, 1.0), (500, 40, 60, 12, 0.2),
                                                  (128, 1, 3, 6, 1.0), (300, 30, 30, 5, 0.0)):
    cur = set(rng.choice(n_pages, per_step, replace=False).tolist())
    traces = []
    for _ in range(steps):
        keep = [p for p in sorted(cur) if rng.random() > churn]
        pool = [p for p in range(n_pages) if p not in keep]
        new = rng.choice(pool, per_step - len(keep), replace=False).tolist() if per_step > len(keep) else []
        cur = set(keep) | set(new)
        traces.append(sorted(int(p) for p in cur))
    cfg = OffloadConfig(layers=1, page_bytes=1, link_bandwidth=1, per_layer_compute=1, fast_tier_capacity=capacity)
    rep = simulate("prefetch", [[t] for t in traces], cfg)
    cases.append({"n_pages": n_pages, "capacity": capacity, "traces": traces,
                  "missing_per_step": [int(c.transfer) for c in rep.steps]})
out = Path(__file__).resolve().parent / "offload_lru.json"
out.write_text(json.dumps({"what": "specsparse.offloadsim.simulate('prefetch') transfers (= missing pages, tau 1) "
                                   "per step for one-layer page traces", "cases": cases}))
print(out, len(cases))
