#!/usr/bin/env python
"""A/B of the single-GPU mode-S select routes on one config: select_kernel (one
CTA per row) vs the chunk-parallel sharded-path select at P = 1.  Times the
select stage (CUDA graph replay, L2 flushed) for both; one JSON line."""
import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2605_15508_b200 import SparsityConfig  # noqa: E402
from paper_2605_15508_b200.verify_step import (STSVerifyStep, config_shape, random_mapping_table,  # noqa: E402
                                          synthetic_inputs)

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--page-size", type=int, default=16)
ap.add_argument("--iters", type=int, default=5)
a = ap.parse_args()
s = config_shape(a.config)
cfg = SparsityConfig(budget=0.1, page_size=a.page_size)
table = random_mapping_table(s, seed=5)
dq, dk, _, _, _ = synthetic_inputs(s, "cuda", seed=0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = {"config": a.config, "page_size": a.page_size}
for name, lr in (("select_kernel", 1 << 30), ("chunk_parallel", 1)):
    step = STSVerifyStep(s, cfg, table, mode="S", long_row_min=lr)
    dqv, dkv = step.draft_views(dq, dk)
    step.capture(dqv, dkv)
    step.build_masks()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step.build_masks()
    ts = []
    for _ in range(a.iters):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    res[name + "_us"] = round(sum(ts) / len(ts), 1)
    res[name + "_cnt0"] = int(step.cnt[0].item())
    del step, g
    torch.cuda.empty_cache()
print(json.dumps(res))
