#!/usr/bin/env python
"""attend_host with the output copied back by the copy engine (D2H after
each unit group) vs written by the attention kernel straight into the pinned
host buffer (direct_out), and the L2 prefetch of the first K/V rows beside
the Q copy (step.l2_prefetch_bytes, MB in the key): time per call as bench.py's e2e measures it, and
equality of the host output with the device-resident attention.

    python tools/e2e_direct_probe.py [c2]
"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2605_15508_b200 import SparsityConfig  # noqa: E402
from paper_2605_15508_b200.verify_step import STSVerifyStep, config_shape, random_mapping_table, synthetic_inputs  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c2"
s = config_shape(cfg_name)
step = STSVerifyStep(s, SparsityConfig(budget=0.1), random_mapping_table(s, 5))
dq, dk, tq, tk, tv = synthetic_inputs(s, "cuda", seed=0)
dqv, dkv = step.draft_views(dq, dk)
step.capture(dqv, dkv)
step.build_masks()
q, k, v = step.target_views(tq, tk, tv)
step.attend(q, k, v)
torch.cuda.synchronize()
ref = step.out.clone()
from bench import L2Flush  # noqa: E402

flush = L2Flush(torch.device("cuda"), "clean")
h_tq = tq.cpu().pin_memory()
res = {"config": cfg_name, "out_bytes": ref.numel() * ref.element_size()}
st = torch.cuda.current_stream()
for direct, chunks, busy, pf_mb in ((False, 2, 0, 0), (True, 1, 0, 0), (True, 1, 0, 16), (True, 1, 0, 32),
                                    (True, 1, 0, 48), (True, 1, 1, 32)):
    step.l2_prefetch_bytes = pf_mb << 20
    if True:
        h_out = torch.zeros(step.out.shape, dtype=step.out.dtype).pin_memory()
        ts = []
        for i in range(25):
            flush()
            if busy:  # keep the GPU busy while the host enqueues: device time only
                torch.cuda._sleep(200000)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            step.attend_host(h_tq, tk, tv, h_out, chunks=chunks, direct_out=direct)
            b.record(st)
            torch.cuda.synchronize()
            if i >= 5:
                ts.append(a.elapsed_time(b) * 1e3)
        ts.sort()
        key = f"{'direct' if direct else 'copy'}_c{chunks}" + ("_busy" if busy else "") + f"_pf{pf_mb}"
        if key + "_us_median" in res:
            key += "_again"
        res[key + "_us_median"] = round(ts[len(ts) // 2], 1)
        res[key + "_us_mean"] = round(sum(ts) / len(ts), 1)
        res[key + "_equal"] = bool(torch.equal(h_out, ref.cpu()))
print(json.dumps(res))
