#!/usr/bin/env python
"""KV offload tier: the target KV cache of
c2 shapes kept in pinned host memory, attention gathered straight over the
host link by the same kernel.  Sparse (90%) vs dense, both offloaded, and the
HBM-resident sparse run for reference.  One JSON line."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2605_15508_b200 import SparsityConfig, kernels  # noqa: E402
from paper_2605_15508_b200.verify_step import (STSVerifyStep, algorithmic_bytes, config_shape,  # noqa: E402
                                          random_mapping_table, synthetic_inputs)

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 8
s = config_shape("c2", target_layers=layers)
step = STSVerifyStep(s, SparsityConfig(budget=0.1), random_mapping_table(s, 5), mode="S")
dq, dk, tq, tk, tv = synthetic_inputs(s, "cuda", seed=0)
q, k, v = step.target_views(tq, tk, tv)
step.capture(*step.draft_views(dq, dk))
step.build_masks()
kh, vh = k.cpu().pin_memory(), v.cpu().pin_memory()
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def timeit(fn, iters=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = ev(), ev()
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / iters


t_dev = timeit(lambda: step.attend(q, k, v), 10)
t_host = timeit(lambda: kernels.sparse_decode(q, kh, vh, idx=step.idx, cnt=step.cnt, causal_base=s.context,
                                              rows_per_head=s.rows, out=step.out, lse=step.lse, host_kv=True))
t_host_dense = timeit(lambda: kernels.sparse_decode(q, kh, vh, n_dense=s.n_kv, causal_base=s.context,
                                                    rows_per_head=s.rows, out=step.out, lse=step.lse,
                                                    host_kv=True), 1)
keys = step.cnt.float().mean().item()
sb, db = algorithmic_bytes(s, keys), algorithmic_bytes(s, s.n_kv, dense=True)
print(json.dumps({
    "workload": f"c2 shapes with {layers} target layers, 32K context, KV in pinned host memory",
    "hbm_sparse_us": round(t_dev, 1), "offload_sparse_us": round(t_host, 1), "offload_dense_us": round(t_host_dense, 1),
    "offload_sparse_vs_dense": round(t_host_dense / t_host, 2), "offload_over_hbm": round(t_host / t_dev, 1),
    "host_link_GBps_sparse": round(sb / (t_host * 1e-6) / 1e9, 1), "host_link_GBps_dense": round(db / (t_host_dense * 1e-6) / 1e9, 1),
    "sparse_bytes": int(sb), "dense_bytes": int(db)}))
