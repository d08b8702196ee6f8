#!/usr/bin/env python
"""Small invocations of every kernel family of libsts_b200.so, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck) runs
(tests/test_gpu_sanitizer.py).  No parity checks here: the tools report
hazards; the parity suite checks values."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2605_15508_b200 import SparsityConfig, kernels  # noqa: E402
from paper_2605_15508_b200.model import block_attention  # noqa: E402
from paper_2605_15508_b200.sharded import DistSelector, run_single  # noqa: E402
from paper_2605_15508_b200.verify_step import STSVerifyStep, VerifyShape, random_mapping_table, synthetic_inputs  # noqa: E402

which = set(sys.argv[1:]) or {"capture", "select", "decode", "dist", "merge", "prefill", "block", "union",
                              "prefill_tc", "offload"}
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
s = VerifyShape(batch=1, context=1000, gamma=4, target_layers=2, target_q_heads=8, target_kv_heads=2, head_dim=128,
                draft_layers=2, draft_q_heads=8, draft_kv_heads=2, draft_head_dim=64)
dq, dk, tq, tk, tv = synthetic_inputs(s, dev, seed=0)
cfg = SparsityConfig(budget=0.1)
if "capture" in which or "select" in which or "decode" in which:
    for mode in ("S", "R"):
        step = STSVerifyStep(s, cfg, random_mapping_table(s, 1), mode=mode, device=dev)
        q, k, v = step.target_views(tq, tk, tv)
        dqv, dkv = step.draft_views(dq, dk)
        step.capture(dqv, dkv)
        step.build_masks()
        for sched in ((0, 1, 2, 3) if mode == "S" else (0,)):
            step.schedule = sched
            step.attend(q, k, v)
        step.attend_dense(q, k, v)
    kernels.draft_scores(dqv, dkv, G=s.draft_group, R=s.rows, base=s.context)
if "select" in which:
    rows = torch.rand((6, 2048), generator=g, device=dev)
    for ps in (1, 16):
        kernels.select_topk(rows, budget=0.1, page_size=ps, row_len=torch.full((6,), 1500, dtype=torch.int32, device=dev),
                            include_sink=True, recent_window=4)
    # register kernel at 32K keys (4-source group sums, tie-heavy rows -> ranked ties across warps)
    coarse = torch.floor(torch.rand((4, 32776), generator=g, device=dev) * 4) / 4
    src = torch.tensor([[0, 1, 2, 3], [3, 2, 1, 0]], dtype=torch.int32, device=dev)
    kernels.select_topk(coarse, budget=3277, row_src=src, n_common=32768, include_current=False, tail_len=5)
if "dist" in which:
    n = 70001
    rows = torch.rand((3, -(-n // 4) * 4), generator=g, device=dev)
    sel = DistSelector(3, n, 1, 1, dev)
    idx = torch.empty((3, 8000), dtype=torch.int32, device=dev)
    cnt = torch.empty((3,), dtype=torch.int32, device=dev)
    st = torch.zeros((1,), dtype=torch.int32, device=dev)
    run_single(sel.protocol(rows, row_src=None, n_global=n - 5, lo=0, k_top=700, rank=0, include_current=False,
                            include_sink=False, recent_window=0, tail_len=5, n_kv_local=n, idx=idx, cnt=cnt, status=st))
if "merge" in which:
    o = torch.randn((3, 40, 128), generator=g, device=dev)
    l = torch.randn((3, 40), generator=g, device=dev)
    kernels.lse_merge(o, l)
if "prefill" in which:
    n = 96
    q = torch.randn((2, n, 4, 128), generator=g, device=dev).bfloat16()
    kk = torch.randn((2, n, 128), generator=g, device=dev).bfloat16()
    vv = torch.randn((2, n, 128), generator=g, device=dev).bfloat16()
    idx = torch.zeros((2 * n, n), dtype=torch.int32, device=dev)
    cnt = torch.zeros((2 * n,), dtype=torch.int32, device=dev)
    for r in range(2 * n):
        t = r % n
        m = np.unique(np.concatenate([np.arange(0, t + 1, 3), [t]]))
        idx[r, : m.size] = torch.from_numpy(m.astype(np.int32))
        cnt[r] = m.size
    kernels.sparse_prefill(q, kk, vv, idx=idx, cnt=cnt)
    # L2 prefetch of K/V rows (the host-buffer verify step): idx / cnt reads
    kernels.kv_prefetch_l2(kk, vv, idx=idx[::n].contiguous(), cnt=cnt[::n].contiguous(), parts=3, keys_per_part=8)
if "block" in which:
    H, m, d, start = 3, 4, 16, 40
    kk = torch.randn((H, start + m, d), generator=g, device=dev)
    block_attention(torch.randn((H, m, d), generator=g, device=dev), kk, kk.clone(), start, record_attention=True,
                    record_scores=True)
if "union" in which:
    idx = torch.sort(torch.randint(0, 500, (8, 60), generator=g, device=dev, dtype=torch.int32), dim=1).values
    cnt = torch.full((8,), 60, dtype=torch.int32, device=dev)
    kernels.row_union(idx, cnt, torch.arange(8, dtype=torch.int32, device=dev).reshape(2, 4), M=4, n_max=500)
if "prefill_tc" in which:
    # 300 tokens: one item per CTA; 2600 tokens x 8 heads = 168 items > the SMs,
    # so persistent CTAs also run items back to back
    for n, hq, hkv, d in ((300, 2, 1, 128), (2600, 8, 2, 128)):
        q = torch.randn((hq, n, d), generator=g, device=dev).bfloat16()
        kk = torch.randn((hkv, n, d), generator=g, device=dev).bfloat16()
        vv = torch.randn((hkv, n, d), generator=g, device=dev).bfloat16()
        tiles = -(-n // 128)
        sc = torch.rand((hkv * tiles, -(-n // 4) * 4), generator=g, device=dev)
        idx, cnt = kernels.prefill_tile_select(sc, budget=0.3, n=n)
        kernels.prefill_blocksparse(q, kk, vv, idx=idx, cnt=cnt)
        kernels.prefill_blocksparse(q, kk, vv)
if "offload" in which:
    from paper_2605_15508_b200.offload import PagedKVOffload

    step = STSVerifyStep(s, SparsityConfig(budget=0.1, page_size=16), random_mapping_table(s, 1), mode="S",
                         device=dev)
    q, k, v = step.target_views(tq, tk, tv)
    step.capture(*step.draft_views(dq, dk))
    step.build_masks()
    off = PagedKVOffload(step, k.cpu().pin_memory(), v.cpu().pin_memory(), page_size=16, copy_ctas=4)
    off.attend_on_demand(q)
    off.attend_prefetch(q)
torch.cuda.synchronize()
print("sanitize_run ok:", ",".join(sorted(which)))
