#!/usr/bin/env python
"""Gather roofline probe (tuning aid): HBM read rate of a pure gather of the
c2 mode-S selection (K and V rows of every selected key, no math) beside the
attention kernel on the same lists, and a dense streaming read of the whole
K/V.  Needs tools/_build/gather_probe.so (built by `python tools/gather_probe.py --build`)."""
import ctypes
import json
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
SO = HERE / "_build" / "gather_probe.so"
if "--build" in sys.argv:
    SO.parent.mkdir(exist_ok=True)
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                    "-o", str(SO), str(HERE / "gather_probe.cu")], check=True)
    sys.exit(0)

import torch  # noqa: E402

sys.path.insert(0, str(HERE.parent))
from paper_2605_15508_b200 import SparsityConfig  # noqa: E402
from paper_2605_15508_b200.verify_step import (STSVerifyStep, algorithmic_bytes, config_shape,  # noqa: E402
                                               random_mapping_table, synthetic_inputs)

lib = ctypes.CDLL(str(SO))
lib.gather_probe.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_longlong] * 2 + [ctypes.c_int] * 6 + [ctypes.c_void_p] * 2
import argparse  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--sparsity", type=float, default=0.9)
a = ap.parse_args([x for x in sys.argv[1:] if x != "--build"])
s = config_shape(a.config)
step = STSVerifyStep(s, SparsityConfig(budget=round(1 - a.sparsity, 6)), random_mapping_table(s, 5), mode="S",
                     device="cuda")
dq, dk, tq, tk, tv = synthetic_inputs(s, "cuda", seed=0)
q, k, v = step.target_views(tq, tk, tv)
dqv, dkv = step.draft_views(dq, dk)
step.step(dqv, dkv, q, k, v)
torch.cuda.synchronize()
U = k.shape[0]
out = torch.zeros(U * 64, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
acc = torch.empty((), dtype=torch.int64, device="cuda")


def clean_flush():  # as bench.py's L2Flush("clean"): write, then read back (no dirty lines left)
    flush.zero_()
    torch.sum(flush.view(-1, 8).view(torch.int64), dim=(0, 1), out=acc)

st = torch.cuda.current_stream().cuda_stream
row_vecs = s.head_dim * 2 // 16


def timed(fn, iters=20):
    ts = []
    for _ in range(iters):
        clean_flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


keys = float(step.cnt.sum().item())
res = {"workload": f"{a.config} mode S {a.sparsity:g}", "rows_per_unit": int(step.M), "selected_keys": int(keys),
       "peak_copy_gbs": 6549.4}
def probe(splits, unroll, dense_n=0, key_stride=1):
    return timed(lambda: lib.gather_probe(k.data_ptr(), v.data_ptr(), step.idx.data_ptr(), step.cnt.data_ptr(),
                                          step.idx.stride(0), k.stride(0) * 2 // 16, row_vecs, U, splits, dense_n,
                                          key_stride, unroll, out.data_ptr(), st))


row_bytes = 2 * s.head_dim * 2  # K + V row
for splits in (4, 8, 16):
    for unroll in (4, 16):
        t = probe(splits, unroll)
        res[f"gather_us_s{splits}_u{unroll}"] = round(t, 2)
        res[f"gather_gbs_s{splits}_u{unroll}"] = round(keys * row_bytes / t / 1e3, 1)
n = s.n_kv
t = probe(16, 4, n)
res["dense_read_us"] = round(t, 2)
res["dense_read_gbs"] = round(U * n * row_bytes / t / 1e3, 1)
per_unit = int(keys // U)
t = probe(16, 4, per_unit, n // per_unit)
res["stride_read_us"] = round(t, 2)
res["stride_read_gbs"] = round(U * per_unit * row_bytes / t / 1e3, 1)
res["stride_keys"] = n // per_unit
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    step.attend(q, k, v)
t = timed(g.replay)
res["attend_us"] = round(t, 2)
ab = algorithmic_bytes(s, keys / U)
res["attend_algorithmic_gbs"] = round(ab / t / 1e3, 1)
print(json.dumps(res))
