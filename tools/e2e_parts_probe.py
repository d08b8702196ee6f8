"""Components of the host-buffer e2e at c2, each as its own CUDA graph with the
bench's L2 flush: device attention, attention writing the pinned host output,
H2D of the target Q, D2H of the output."""
import json, sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2605_15508_b200 import SparsityConfig
from paper_2605_15508_b200.verify_step import STSVerifyStep, config_shape, random_mapping_table, synthetic_inputs
from bench import L2Flush
s = config_shape("c2")
step = STSVerifyStep(s, SparsityConfig(budget=0.1), random_mapping_table(s, 5))
dq, dk, tq, tk, tv = synthetic_inputs(s, "cuda", seed=0)
step.capture(*step.draft_views(dq, dk)); step.build_masks()
q, k, v = step.target_views(tq, tk, tv)
h_tq = tq.cpu().pin_memory()
h_out = torch.empty(step.out.shape, dtype=step.out.dtype).pin_memory()
_, d_tq = step._host_buffers(None, h_tq)
d_tq.copy_(tq)
qd, _, _ = step.target_views(d_tq, tk, tv)
flush = L2Flush(torch.device("cuda"), "clean")
st = torch.cuda.current_stream()
def t(fn, n=25):
    g = step._graph(("probe", id(fn)), fn)
    ts = []
    for i in range(n):
        flush(); a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); g.replay(); b.record(st); torch.cuda.synchronize()
        if i >= 5: ts.append(a.elapsed_time(b) * 1e3)
    ts.sort(); return round(ts[len(ts)//2], 1)
f_dev = lambda: step.attend(qd, tk.flatten(0, 2) if tk.dim() == 5 else tk, tv.flatten(0, 2) if tv.dim() == 5 else tv)
f_dev = lambda: step._attend_pipelined(None, d_tq, qd, *step.target_views(d_tq, tk, tv)[1:], step.out, 1)
f_dout = lambda: step._attend_pipelined(None, d_tq, qd, *step.target_views(d_tq, tk, tv)[1:], h_out, 1, direct_out=True)
f_h2d = lambda: d_tq.copy_(h_tq, non_blocking=True)
f_d2h = lambda: h_out.copy_(step.out, non_blocking=True)
print(json.dumps({"attend_device_us": t(f_dev), "attend_direct_out_us": t(f_dout), "h2d_q_us": t(f_h2d), "d2h_out_us": t(f_d2h)}))
