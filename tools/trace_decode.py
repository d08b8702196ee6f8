#!/usr/bin/env python
"""Per-CTA timeline of the verify decode kernel (needs the STS_TRACE variant:
STS_B200_LIB=.../libsts_b200_trace.so).  Runs the c2 sparse decode a few times
and prints the distribution of entry / first-data / loop-end / exit times."""
import ctypes
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2605_15508_b200 import SparsityConfig, _lib  # noqa: E402
from paper_2605_15508_b200.verify_step import STSVerifyStep, config_shape, random_mapping_table, synthetic_inputs  # noqa: E402

ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
lib = _lib.load()
lib.sts_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
s = config_shape("c2", context=ctx)
step = STSVerifyStep(s, SparsityConfig(budget=0.1), random_mapping_table(s, 5), mode="S", device="cuda")
dq, dk, tq, tk, tv = synthetic_inputs(s, "cuda", seed=0)
q, k, v = step.target_views(tq, tk, tv)
dqv, dkv = step.draft_views(dq, dk)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    step.step(dqv, dkv, q, k, v)
torch.cuda.synchronize()
out = {}
for name, fn in (("sparse", lambda: step.attend(q, k, v)), ("dense", lambda: step.attend_dense(q, k, v))):
    flush.zero_()
    flush.sum()
    torch.cuda.synchronize()
    fn()
    torch.cuda.synchronize()
    buf = np.zeros(8192 * 8, dtype=np.uint64)
    assert lib.sts_debug_trace(buf.ctypes.data, buf.nbytes) == 0
    t = buf.reshape(8192, 8).astype(np.float64)
    live = t[:, 0] > 0
    t = t[live]
    t0 = t[:, 0].min()
    rel = (t[:, :5] - t0) / 1e3  # us
    pct = lambda x: [round(float(np.percentile(x, q)), 2) for q in (0, 10, 50, 90, 100)]  # noqa: E731
    out[name] = {"ctas": int(live.sum()), "entry": pct(rel[:, 0]), "first_issue": pct(rel[:, 1]),
                 "first_tile": pct(rel[:, 2]), "loop_end": pct(rel[:, 3]), "exit": pct(rel[:, 4]),
                 "flush_us_per_cta": pct(t[:, 5] / 1e3), "flushes": pct(t[:, 6]),
                 "tiles": pct(buf.reshape(8192, 8)[live, 7] & 0xffffffff)}
    sm = (buf.reshape(8192, 8)[live, 7] >> 32).astype(np.int64)
    per_sm = np.zeros(sm.max() + 1)
    for smi, le in zip(sm, rel[:, 3]):
        per_sm[smi] = max(per_sm[smi], le)
    order = np.argsort(per_sm)
    out[name]["slowest_sms_loop_end"] = [(int(i), round(float(per_sm[i]), 1)) for i in order[-12:]]
    out[name]["fastest_sms_loop_end"] = [(int(i), round(float(per_sm[i]), 1)) for i in order[:12]]
    # spread of loop-end within an SM vs across SMs
    within = []
    for smi in np.unique(sm):
        le_s = rel[sm == smi, 3]
        within.append(le_s.max() - le_s.min())
    out[name]["within_sm_spread_us"] = pct(np.array(within))
print(json.dumps(out, indent=1))
