#!/usr/bin/env python
"""Algorithm 1 overlap kernel at real head counts (one B200): Ta target heads x
Tb draft heads, n rows of n-bit top-k sets per head (W = n * n/32 words).
Reports the sts_bitset_overlap time and its AND+popcount rate.  One JSON line."""
import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2605_15508_b200 import _lib  # noqa: E402
from paper_2605_15508_b200._lib import call, ptr, stream_handle  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ta", type=int, default=1024)
ap.add_argument("--tb", type=int, default=512)
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
_lib.load()
W = a.n * (a.n // 32)
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randint(-2**31, 2**31 - 1, (a.ta, W), generator=g, device="cuda", dtype=torch.int32)
B = torch.randint(-2**31, 2**31 - 1, (a.tb, W), generator=g, device="cuda", dtype=torch.int32)
S = torch.zeros((a.ta, a.tb), dtype=torch.int64, device="cuda")
run = lambda: call("sts_bitset_overlap", ptr(A), a.ta, ptr(B), a.tb, W, ptr(S), stream_handle())  # noqa: E731
run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.iters):
    run()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.iters
words = a.ta * a.tb * W
print(json.dumps({"workload": f"Algorithm 1 overlap: {a.ta} target x {a.tb} draft heads, {a.n} rows x {a.n} bits",
                  "ms": round(ms, 3), "word_pairs_per_s": f"{words / (ms * 1e-3):.3e}",
                  "bit_ops_per_s": f"{32 * words / (ms * 1e-3):.3e}"}))
