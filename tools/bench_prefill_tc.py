#!/usr/bin/env python
"""Block-sparse prefill on tcgen05 vs dense prefill on one
B200: one Llama-3.1-8B layer (32 q-heads, 8 kv-heads, d=128), prompt n,
90% sparsity (budget 0.1 of each tile's committed context, 64-key blocks,
128-row query tiles).  Reports the block selection (GPU select over the
per-(kv-head, tile) draft score rows), the sparse attention, the same kernel
dense (all blocks), and flash_attn's dense causal prefill (library, sanity
bar).  One JSON line per n."""
import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2605_15508_b200 import kernels  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, nargs="+", default=[4096, 16384, 32768])
ap.add_argument("--iters", type=int, default=10)
a = ap.parse_args()
Hq, Hkv, d = 32, 8, 128
dev = torch.device("cuda")
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


for n in a.n:
    g = torch.Generator(device=dev).manual_seed(0)
    q = torch.randn((Hq, n, d), generator=g, device=dev).bfloat16()
    k = torch.randn((Hkv, n, d), generator=g, device=dev).bfloat16()
    v = torch.randn((Hkv, n, d), generator=g, device=dev).bfloat16()
    tiles = -(-n // 128)
    scores = torch.softmax(2 * torch.randn((Hkv * tiles, -(-n // 4) * 4), generator=g, device=dev), -1).contiguous()
    sel = {}
    t_sel = timeit(lambda: sel.update(zip(("idx", "cnt"), kernels.prefill_tile_select(scores, budget=0.1, n=n))))
    # the same selection replayed as a CUDA graph (no host launch gaps)
    gsel = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gsel):
        gi, gc = kernels.prefill_tile_select(scores, budget=0.1, n=n)
    t_sel_graph = timeit(gsel.replay)
    out = torch.empty_like(q)
    t_sp = timeit(lambda: kernels.prefill_blocksparse(q, k, v, idx=sel["idx"], cnt=sel["cnt"], out=out))
    t_dn = timeit(lambda: kernels.prefill_blocksparse(q, k, v, out=out))
    blocks = float(sel["cnt"].sum().item()) / 64 + Hkv * (2 * tiles - 0.5)
    dense_blocks = Hkv * sum(2 * T + 2 for T in range(tiles))
    flops_dense = 4.0 * Hq * d * sum(min(128 * T + 128, n) * 128 - 64 * 127 for T in range(tiles))
    line = {"workload": f"block-sparse prefill, one Llama-3.1-8B layer (32 q / 8 kv heads, d=128), n={n}, "
                        "budget 0.1 per 128-row tile, 64-key blocks",
            "tile_select_us": round(t_sel, 1), "tile_select_graph_us": round(t_sel_graph, 1),
            "sparse_prefill_us": round(t_sp, 1),
            "sparse_incl_select_us": round(t_sel + t_sp, 1), "dense_same_kernel_us": round(t_dn, 1),
            "block_fraction": round(blocks / dense_blocks, 3),
            "dense_same_kernel_TFLOPs": round(flops_dense / (t_dn * 1e-6) / 1e12, 1)}
    try:
        from flash_attn import flash_attn_func

        qd = q.permute(1, 0, 2).unsqueeze(0).contiguous()   # [1, n, Hq, d]
        kd = k.permute(1, 0, 2).unsqueeze(0).contiguous()
        vd = v.permute(1, 0, 2).unsqueeze(0).contiguous()
        t_fa = timeit(lambda: flash_attn_func(qd, kd, vd, causal=True))
        line["dense_flash_attn_us"] = round(t_fa, 1)
        line["speedup_vs_flash_attn_incl_select"] = round(t_fa / (t_sel + t_sp), 2)
    except Exception as exc:  # pragma: no cover
        line["dense_flash_attn_us"] = f"unavailable: {exc}"[:120]
    line["speedup_vs_dense_same_kernel"] = round(t_dn / t_sp, 2)
    print(json.dumps(line), flush=True)
