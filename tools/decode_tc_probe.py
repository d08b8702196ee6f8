#!/usr/bin/env python
"""tcgen05-versus-mma.sync comparison for the gathered verify decode (tuning
aid): runs the prototype tools/decode_tc.cu (keys as M = 128 in
TMEM lanes, the unit's rows as N = 48) and the library's mma.sync decode on
the same mode-S step, checks they agree (bf16 tolerance) and times both
(clean L2 flush, median of 20).  One JSON line per config.

    python tools/decode_tc_probe.py --build
    python tools/decode_tc_probe.py --config c3 --sparsity 0.9
"""
import argparse
import ctypes
import json
import math
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
import os
SO = Path(os.environ.get("DECODE_TC_SO", str(HERE / "_build" / "decode_tc.so")))
if "--build" in sys.argv:
    SO.parent.mkdir(exist_ok=True)
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared", "-Xcompiler",
                    "-fPIC", "-I", str(HERE.parent / "paper_2605_15508_b200" / "csrc"), "-o", str(SO),
                    str(HERE / "decode_tc.cu")], check=True)
    sys.exit(0)

import torch  # noqa: E402

sys.path.insert(0, str(HERE.parent))
from paper_2605_15508_b200 import SparsityConfig  # noqa: E402
from paper_2605_15508_b200.verify_step import (STSVerifyStep, VerifyShape, config_shape,  # noqa: E402
                                               random_mapping_table, synthetic_inputs)

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--sparsity", type=float, default=0.9)
ap.add_argument("--context", type=int, default=None)
a = ap.parse_args()
lib = ctypes.CDLL(str(SO))
lib.decode_tc.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_longlong] * 2 + [ctypes.c_int] * 3 + \
    [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p, ctypes.c_float, ctypes.c_void_p, ctypes.c_void_p,
     ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
if a.config == "small":
    s = VerifyShape(batch=2, context=5000, gamma=4, target_layers=3, target_q_heads=14, target_kv_heads=2,
                    head_dim=128, draft_layers=2, draft_q_heads=8, draft_kv_heads=2, draft_head_dim=64)
else:
    s = config_shape(a.config, **({"context": a.context} if a.context else {}))
step = STSVerifyStep(s, SparsityConfig(budget=round(1 - a.sparsity, 6)), random_mapping_table(s, 5), mode="S",
                     device="cuda")
dq, dk, tq, tk, tv = synthetic_inputs(s, "cuda", seed=0)
q, k, v = step.target_views(tq, tk, tv)
step.capture(*step.draft_views(dq, dk))
step.build_masks()
torch.cuda.synchronize()
U, M = k.shape[0], step.M
out_tc = torch.empty_like(step.out)
lse_tc = torch.empty_like(step.lse)
sms = torch.cuda.get_device_properties(0).multi_processor_count
st = torch.cuda.current_stream().cuda_stream
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
acc = torch.empty((), dtype=torch.int64, device="cuda")


dbg = torch.zeros(16, dtype=torch.int64, device="cuda")


def run_tc(d=None):
    rc = lib.decode_tc(q.data_ptr(), k.data_ptr(), v.data_ptr(), k.stride(0), U, M, s.rows, s.context,
                       step.idx.data_ptr(), step.idx.stride(0), step.cnt.data_ptr(), 1.0 / math.sqrt(s.head_dim),
                       out_tc.data_ptr(), lse_tc.data_ptr(), sms, st, d.data_ptr() if d is not None else None)
    assert rc == 0, rc


def timed(fn, iters=20):
    ts = []
    for _ in range(iters):
        flush.zero_()
        torch.sum(flush.view(-1, 8).view(torch.int64), dim=(0, 1), out=acc)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


step.attend(q, k, v)
run_tc(dbg)
torch.cuda.synchronize()
cyc = dbg.cpu().tolist()
tiles = max(1, cyc[3])
cycles = {"tiles_cta0": cyc[3]} | {name: round(cyc[i] / tiles) for i, name in enumerate(
    ["sm_wait_S", "sm_compute", "sm_wait_Pbuf", None, "mma_wait_Sslot", "mma_wait_K", "mma_wait_P", "mma_wait_O",
     "mma_wait_V"]) if name}
diff = (out_tc.float() - step.out.float()).abs().max().item()
lse_diff = (lse_tc - step.lse).abs().max().item()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    step.attend(q, k, v)
t_mma = timed(g.replay)
t_tc = timed(run_tc)
print(json.dumps({"config": a.config, "sparsity": a.sparsity, "rows_per_unit": M, "units": U,
                  "keys_per_unit": round(step.cnt.float().mean().item(), 1),
                  "mma_sync_us": round(t_mma, 1), "tcgen05_prototype_us": round(t_tc, 1),
                  "max_abs_diff_out": diff, "max_abs_diff_lse": lse_diff, "cycles_per_tile_cta0": cycles}))
