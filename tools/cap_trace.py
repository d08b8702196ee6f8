#!/usr/bin/env python
"""Per-role cycle accounting of the capture kernel (needs the STS_CAP_TRACE
variant: build_variant("trace", ["STS_CAP_TRACE"]); run with
STS_B200_LIB=paper_2605_15508_b200/_lib/variants/libsts_b200_trace.so)."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2605_15508_b200 import SparsityConfig, _lib  # noqa: E402
from paper_2605_15508_b200.verify_step import STSVerifyStep, config_shape, random_mapping_table, synthetic_inputs  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c2"
lib = _lib.load()
lib.sts_cap_trace.argtypes = [C.c_void_p, C.c_int]
s = config_shape(cfg_name)
step = STSVerifyStep(s, SparsityConfig(budget=0.1), random_mapping_table(s, 5))
dq, dk, tq, tk, tv = synthetic_inputs(s, "cuda", seed=0)
dqv, dkv = step.draft_views(dq, dk)
for _ in range(2):
    step.capture(dqv, dkv)
torch.cuda.synchronize()
for name, fn in (("lse", lambda: __import__("paper_2605_15508_b200.kernels", fromlist=["x"]).draft_lse(
        dqv, dkv, G=s.draft_group, R=s.rows, base=s.context, n_keys=s.n_kv, out=step.draft_lse, workspace=step.ws_draft)),
                 ("capture(lse+probs)", lambda: step.capture(dqv, dkv))):
    lib.sts_cap_trace(None, 1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    buf = np.zeros(1024 * 16 * 4, dtype=np.uint64)
    lib.sts_cap_trace(buf.ctypes.data, 0)
    t = buf.reshape(1024, 16, 4)[:148].astype(np.float64)
    print(f"== {name}: {e0.elapsed_time(e1) * 1e3:.1f} us")
    for w, role in ((0, "producer (wait empty)"), (1, "mma (wait acce | wait full)")):
        tiles = t[:, w, 3].sum()
        print(f"  {role}: tiles {tiles:.0f}, wait0/tile {t[:, w, 0].sum() / tiles:.0f} cyc, wait1/tile {t[:, w, 1].sum() / tiles:.0f} cyc, total/cta {t[:, w, 2].mean():.0f} cyc")
    for w in range(2, 10):
        tiles = t[:, w, 3].sum()
        if tiles == 0:
            continue
        print(f"  epi warp {w}: tiles {tiles:.0f}, wait accf/tile {t[:, w, 0].sum() / tiles:.0f} cyc, ld/tile {t[:, w, 1].sum() / tiles:.0f} cyc, total/cta {t[:, w, 2].mean():.0f} cyc")
