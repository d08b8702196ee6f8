#!/usr/bin/env python
"""Sparse prefill (STS-PD) timing on one B200: one target layer of Llama-3.1-8B
shapes (8 kv-heads x 4 q-heads sharing a row mask, d = 128), prompt n, 90%
sparsity per row (budget 0.1 of each causal prefix + current).  Reports the
mask build (GPU select over the n draft rows per kv-head), the sparse prefill
attention, and a dense causal prefill (flash_attn, library, sanity bar) for
the same layer.  One JSON line."""
import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2605_15508_b200 import kernels  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=4096)
ap.add_argument("--iters", type=int, default=10)
a = ap.parse_args()
n, G, M, d = a.n, 8, 4, 128
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
logits = 2.0 * torch.randn((G * n, n), generator=g, device=dev)
causal = torch.arange(n, device=dev)[None, :] <= torch.arange(n, device=dev).repeat(G)[:, None]
rows = torch.softmax(logits.masked_fill(~causal, float("-inf")), dim=-1).float().contiguous()
row_len = torch.arange(1, n + 1, dtype=torch.int32, device=dev).repeat(G)
q = torch.randn((G, n, M, d), generator=g, device=dev).bfloat16()
k = torch.randn((G, n, d), generator=g, device=dev).bfloat16()
v = torch.randn((G, n, d), generator=g, device=dev).bfloat16()
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def timeit(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = ev(), ev()
    e0.record()
    for _ in range(a.iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / a.iters


sel = {}
t_sel = timeit(lambda: sel.update(zip(("idx", "cnt"), kernels.select_topk(rows, row_len=row_len, budget=0.1))))
t_att = timeit(lambda: kernels.sparse_prefill(q, k, v, idx=sel["idx"], cnt=sel["cnt"]))
keys = float(sel["cnt"].float().sum().item())
line = {"workload": f"sparse prefill, one Llama-3.1-8B layer (8 kv x 4 q heads, d=128), n={n}, budget 0.1/row",
        "select_us": round(t_sel, 1), "sparse_prefill_us": round(t_att, 1), "keys_total": int(keys),
        "gathered_GB": round(keys * d * 2 * 2 / 1e9, 3)}
try:
    from flash_attn import flash_attn_func

    qd = q.permute(0, 2, 1, 3).reshape(1, G * M, n, d).transpose(1, 2).contiguous()   # [1, n, Hq, d]
    kd = k.permute(1, 0, 2).unsqueeze(0).contiguous()                                 # [1, n, Hkv, d]
    vd = v.permute(1, 0, 2).unsqueeze(0).contiguous()
    line["dense_flash_attn_us"] = round(timeit(lambda: flash_attn_func(qd, kd, vd, causal=True)), 1)
except Exception as exc:  # pragma: no cover
    line["dense_flash_attn_us"] = f"unavailable: {exc}"[:120]
print(json.dumps(line))
