#!/usr/bin/env python
"""STS verify-step benchmark on B200 (driver contract: one JSON line on rank 0).

Metric (BASELINE.json): target-attention µs per verify step at 90% sparsity,
with speedup vs a dense decode on the same GPU and achieved HBM GB/s.

  python bench.py [--gpus 1] [--steps 20] [--warmup 5] [--config c2] [--mode S]
  python bench.py --impl reference ...   # the reference CPU path (oracle port)

Workload at N=1: BASELINE config 2 — Llama-3.2-1B draft -> Llama-3.1-8B target
shapes, 32K context, batch 1, 90% sparsity, gamma=4 (5 stacked rows x GQA 4),
synthetic N(0,1) bf16 Q/K/V, random head mapping.  A "step" is one verify
step: draft-score capture, mask build, sparse target attention over all 32
layers x 8 kv-heads.  ``value`` is the sparse target-attention time of the
step (inputs resident in HBM, L2 flushed before every timed iteration); the
capture / select stages, the dense decode and the end-to-end public-API time
(host->device Q copies and the device->host output copy included) are
reported beside it.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "target attn us/verify step at 90% sparsity; speedup vs dense; HBM GB/s"
MODEL_NAMES = {
    "c1": "tiny draft 2L/4H -> target 4L/8H",
    "c2": "Llama-3.2-1B draft -> Llama-3.1-8B target",
    "c3": "Qwen2.5-0.5B draft -> Qwen2.5-7B target",
    "c4": "Llama-3.2-1B draft -> Llama-3.1-8B target",
    "c5": "Llama-3.2-1B draft -> Llama-3.1-70B target",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="auto",
                    help="auto = c2 on one GPU, c4 (1M context, KV sharded by sequence) when --gpus > 1")
    ap.add_argument("--mode", default="S", choices=["S", "R"])
    ap.add_argument("--sparsity", type=float, default=0.9)
    ap.add_argument("--page-size", type=int, default=1)
    ap.add_argument("--layout", default="separate", choices=["separate", "interleaved"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="bound of the CPU baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--eager", action="store_true", help="time stages as eager launches instead of CUDA graphs")
    ap.add_argument("--flush", default="clean", choices=["clean", "write", "none"], help="L2 flush between stages")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="collective backend for N > 1 (gloo + --one-gpu: functional check on a single GPU)")
    ap.add_argument("--one-gpu", action="store_true", help="map every rank to cuda:0 (functional checks only)")
    ap.add_argument("--head-groups", type=int, default=0,
                    help="heads x sequence sharding: ranks per head group = gpus / head_groups (0: 2 for c5, else 1)")
    ap.add_argument("--merge", default="gather", choices=["gather", "p2p"],
                    help="sharded path: NCCL all-gather + merge, or one peer-memory merge kernel over symmetric memory")
    ap.add_argument("--context", type=int, default=None, help="override the config's context length")
    ap.add_argument("--batch", type=int, default=None, help="override the config's batch")
    return ap.parse_args()


def shape_overrides(args):
    o = {}
    if args.context is not None:
        o["context"] = args.context
    if args.batch is not None:
        o["batch"] = args.batch
    return o


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class L2Flush:
    """Evict L2 (126 MB) between timed stages with a 256 MB buffer.

    "write": zero the buffer (leaves ~126 MB of dirty lines that the next
    kernel's reads must write back); "clean": zero it and then read it back
    (the L2 ends full of clean, useless lines — the timed kernel starts cold
    without inheriting the flush's write-back traffic); "none": no flush.
    """

    def __init__(self, dev, mode="clean"):
        import torch

        self.mode = mode
        self.buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if mode != "none" else None
        self.acc = torch.empty((), dtype=torch.int64, device=dev) if mode == "clean" else None

    def __call__(self):
        import torch

        if self.mode == "none":
            return
        self.buf.zero_()
        if self.mode == "clean":
            torch.sum(self.buf.view(-1, 8).view(torch.int64), dim=(0, 1), out=self.acc)

    def describe(self):
        return {"write": "flushed by a 256 MB write before every timed stage",
                "clean": "flushed by a 256 MB write + read-back (clean eviction) before every timed stage",
                "none": "not flushed (inputs larger than L2)"}[self.mode]


class ClockSampler:
    """Samples SM clock + throttle reasons through NVML while the timed loop runs."""

    def __init__(self, index=0, period=0.05):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.period, self.index = period, index
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.nv = pynvml
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception as exc:  # pragma: no cover - NVML missing
            self.error = str(exc)
        return self

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        s = sorted(self.samples)
        med = s[len(s) // 2] if s else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(s)}


# ---------------------------------------------------------------------------
# CPU reference path (oracle port of specsparse.sparsity.sparse_attention)
# ---------------------------------------------------------------------------

def _cpu_call_worker(args):
    import numpy as np

    from oracle import sts_oracle as O

    seed, n, d, k = args
    rng = np.random.default_rng(seed)
    q = rng.standard_normal(d).astype(np.float32)
    keys = rng.standard_normal((n, d)).astype(np.float32)
    vals = rng.standard_normal((n, d)).astype(np.float32)
    mask = np.sort(rng.choice(n, size=k, replace=False))
    t0 = time.perf_counter()
    O.sparse_attention(q, keys, vals, mask)
    return time.perf_counter() - t0


def cpu_reference_sample(shape, k_sel, budget_s: float, workers: int):
    """Time oracle sparse_attention calls (one per (layer, head, row) in the
    reference loop) for ~budget_s seconds; return
    (µs per verify step extrapolated, calls timed, per-call seconds)."""
    import multiprocessing as mp

    n, d = shape.n_kv, shape.head_dim
    calls_per_step = shape.batch * shape.target_layers * shape.target_q_heads * shape.rows
    per_call = []
    t_end = time.perf_counter() + budget_s
    seed = 0
    if workers > 1:
        ctx = mp.get_context("fork")
        with ctx.Pool(workers) as pool:
            t0 = time.perf_counter()
            done = 0
            while time.perf_counter() < t_end:
                batch = [(seed + i, n, d, k_sel) for i in range(workers)]
                seed += workers
                per_call.extend(pool.map(_cpu_call_worker, batch))
                done += workers
            wall = time.perf_counter() - t0
        per_call_eff = wall / max(done, 1)  # throughput with `workers` processes
    else:
        while time.perf_counter() < t_end or not per_call:
            per_call.append(_cpu_call_worker((seed, n, d, k_sel)))
            seed += 1
        per_call_eff = sum(per_call) / len(per_call)
    return per_call_eff * calls_per_step * 1e6, len(per_call), per_call_eff


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2605_15508_b200.verify import config_shape

    shape = config_shape(args.config, **shape_overrides(args))
    budget = round(1.0 - args.sparsity, 10)
    k_sel = max(1, math.ceil(budget * (shape.context + 1))) + shape.rows
    workers = os.cpu_count() or 1
    # each call holds K/V in fp32 + their fp64 copies (src/sparsity.py:167-168): ~24 B per element
    per_call_bytes = 24 * shape.n_kv * shape.head_dim
    workers = max(1, min(workers, int(8e9 // per_call_bytes)))
    vals = []
    for i in range(args.warmup + args.steps):
        v, calls, per_call = cpu_reference_sample(shape, k_sel, max(2.0, args.cpu_seconds / max(args.steps, 1)),
                                                  workers)
        if i >= args.warmup:
            vals.append(v)
    value = sum(vals) / len(vals)
    sample = (f"oracle sparse_attention (fp64 numpy, src/sparsity.py:152-173 restated) over n={shape.n_kv}, "
              f"d={shape.head_dim}, |S|={k_sel}; {calls} calls/step-sample on {workers} processes, "
              f"extrapolated x{shape.batch * shape.target_layers * shape.target_q_heads * shape.rows} calls/step")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 1), "unit": "us",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(value / 1e3, 3),
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: target attention of one verify step (CPU reference path)",
                   "sparsity": args.sparsity, "gamma": shape.gamma},
        "cpu_baseline": {"value": round(value, 1), "unit": "us", "cores": workers, "kind": "port", "sample": sample},
        "e2e": {"value": round(value, 1), "unit": "us", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------------------
# GPU path
# ---------------------------------------------------------------------------

def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.config == "auto":
        args.config = "c2" if world == 1 else "c4"
    if args.impl == "reference":
        return run_reference(args)
    if args.config in ("c4", "c5") or world > 1:
        return run_sharded(args, world, rank, local)

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2605_15508_b200 import SparsityConfig, _lib
    from paper_2605_15508_b200.verify import (STSVerifyStep, algorithmic_bytes, config_shape, random_mapping_table,
                                              synthetic_inputs)

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)
    _lib.load()

    shape = config_shape(args.config, **shape_overrides(args))
    budget = round(1.0 - args.sparsity, 10)
    cfg = SparsityConfig(budget=budget, page_size=args.page_size)
    table = random_mapping_table(shape, seed=5 + rank)
    step = STSVerifyStep(shape, cfg, table, mode=args.mode, device=dev)
    dq, dk, tq, tk, tv = synthetic_inputs(shape, dev, seed=100 * rank, layout=args.layout)
    q, k, v = step.target_views(tq, tk, tv)
    dqv, dkv = step.draft_views(dq, dk)
    dense_out = torch.empty_like(step.out)
    dense_lse = torch.empty_like(step.lse)
    flush = L2Flush(dev, args.flush)
    st = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step.step(dqv, dkv, q, k, v)
        step.attend_dense(q, k, v, out=dense_out, lse=dense_lse)
    barrier()
    assert step.status.item() == 0, f"device status {step.status.item()}"

    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    # each stage is captured once into a CUDA graph and replayed, so the
    # device-timed regions hold the kernels only (no Python launch gaps)
    stages = {
        "capture": lambda: step.capture(dqv, dkv),
        "select": lambda: step.build_masks(),
        "attend": lambda: step.attend(q, k, v),
        "dense": lambda: step.attend_dense(q, k, v, out=dense_out, lse=dense_lse),
    }
    run_stage, stage_launches = {}, {}
    lib = _lib.load()
    for name, fn in stages.items():
        c0 = lib.sts_launch_count()
        if args.eager:
            fn()
            run_stage[name] = fn
        else:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                fn()
            run_stage[name] = g.replay
        stage_launches[name] = int(lib.sts_launch_count() - c0)  # our kernels per replay
    for _ in range(2):
        for fn in run_stage.values():
            fn()
    barrier()
    t_cap, t_sel, t_att, t_den = [], [], [], []
    with ClockSampler(local) as clocks:
        barrier()
        wall0 = time.perf_counter()
        for _ in range(args.steps):
            flush()
            e = [ev() for _ in range(4)]
            e[0].record(st)
            run_stage["capture"]()
            e[1].record(st)
            run_stage["select"]()
            e[2].record(st)
            flush()
            e.append(ev())
            e[3].record(st)
            run_stage["attend"]()
            e[4].record(st)
            flush()
            e5, e6 = ev(), ev()
            e5.record(st)
            run_stage["dense"]()
            e6.record(st)
            torch.cuda.synchronize()
            t_cap.append(e[0].elapsed_time(e[1]) * 1e3)
            t_sel.append(e[1].elapsed_time(e[2]) * 1e3)
            t_att.append(e[3].elapsed_time(e[4]) * 1e3)
            t_den.append(e5.elapsed_time(e6) * 1e3)
        barrier()
        wall = time.perf_counter() - wall0

    # end-to-end through the public API with host buffers (pinned), copies inside
    # the timed region: (a) the metric itself — target attention with Q from the
    # host and the output back to the host (STSVerifyStep.attend_host); (b) the
    # whole verify step — capture + select + attention (STSVerifyStep.step_host)
    h_tq = tq.cpu().pin_memory()
    h_dq = dq.cpu().pin_memory()
    h_out = torch.empty(step.out.shape, dtype=step.out.dtype).pin_memory()
    t_e2e, t_e2e_step = [], []
    for i in range(args.warmup + args.steps):
        flush()
        e0, e1 = ev(), ev()
        e0.record(st)
        step.attend_host(h_tq, tk, tv, h_out)
        e1.record(st)
        torch.cuda.synchronize()
        flush()
        e2, e3 = ev(), ev()
        e2.record(st)
        step.step_host(h_dq, dk, h_tq, tk, tv, h_out)
        e3.record(st)
        torch.cuda.synchronize()
        if i >= args.warmup:
            t_e2e.append(e0.elapsed_time(e1) * 1e3)
            t_e2e_step.append(e2.elapsed_time(e3) * 1e3)

    def mean(x):
        return float(sum(x) / len(x))

    stats = torch.tensor([mean(t_att), mean(t_den), mean(t_cap), mean(t_sel), mean(t_e2e), mean(t_e2e_step)],
                         device=dev)
    if world > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.MAX)
    att, den, cap, sel, e2e, e2e_step = stats.tolist()

    cnt = step.cnt.float().mean().item()
    nbytes = algorithmic_bytes(shape, cnt)
    dense_bytes = algorithmic_bytes(shape, shape.n_kv, dense=True)
    peak, peak_src = peaks()
    achieved = nbytes / (att * 1e-6) / 1e9
    traffic = None
    prof = ROOT / "profiles" / "ncu_sparse_decode_summary.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get("dram_bytes_per_step")
        except Exception:
            traffic = None
    launches = args.steps * sum(stage_launches.values())  # counted by the library (sts_launch_count)

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        v_cpu, calls, per_call = cpu_reference_sample(shape, int(round(cnt)), args.cpu_seconds, 1)
        cpu = {"value": round(v_cpu, 1), "unit": "us", "cores": 1, "kind": "port",
               "sample": (f"{calls} oracle sparse_attention calls (fp64 numpy restatement of "
                          f"src/sparsity.py:152-173) at n={shape.n_kv}, d={shape.head_dim}, |S|={int(round(cnt))}, "
                          f"{per_call * 1e3:.1f} ms/call, extrapolated to "
                          f"{shape.batch * shape.target_layers * shape.target_q_heads * shape.rows} calls/step")}

    h2d = tq.numel() * tq.element_size()
    h2d_step = h2d + dq.numel() * dq.element_size()
    d2h = step.out.numel() * step.out.element_size()
    line = {
        "metric": METRIC, "value": round(att, 2), "unit": "us", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(att / 1e3, 5), "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded N(0,1) bf16 Q/K/V, random head mapping)",
        "config": {"workload": f"{args.config}: Llama-3.2-1B draft -> Llama-3.1-8B target shapes, "
                               f"{shape.context} context, batch {shape.batch}, gamma {shape.gamma}, "
                               f"sparsity {args.sparsity}, mode {args.mode}, page_size {args.page_size}, "
                               f"kv layout {args.layout}",
                   "context": shape.context, "batch": shape.batch, "gamma": shape.gamma, "mode": args.mode,
                   "page_size": args.page_size, "kv_layout": args.layout,
                   "keys_per_kv_head": round(cnt, 1), "l2": flush.describe(),
                   "launch": "eager" if args.eager else "CUDA graph per stage",
                   "parallelism": "replicas" if world > 1 else "single"},
        "dense_us": round(den, 2), "speedup_vs_dense": round(den / att, 3),
        "mask_build_us": {"draft_capture": round(cap, 2), "select": round(sel, 2)},
        "sts_step_us": round(cap + sel + att, 2), "step_speedup_vs_dense": round(den / (cap + sel + att), 3),
        "hbm_gbs": round(achieved, 1), "dense_hbm_gbs": round(dense_bytes / (den * 1e-6) / 1e9, 1),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "kernel": "sts_sparse_decode: verify_decode_kernel (gathered flash-decode, cluster/DSMEM or stream-K + piece merge)",
                     "algorithmic_bytes_per_launch": int(nbytes), "peak_source": peak_src},
        "cpu_baseline": cpu,
        "e2e": {"value": round(e2e, 2), "unit": "us", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "what": "public API STSVerifyStep.attend_host: H2D of the target Q from pinned host memory, sparse "
                        "target attention, D2H of the output; one CUDA graph, units in step.host_chunks groups so "
                        "the copies of one group overlap the attention of the other",
                "host_chunks": step.host_chunks},
        "e2e_step": {"value": round(e2e_step, 2), "unit": "us", "h2d_bytes_per_step": int(h2d_step),
                     "d2h_bytes_per_step": int(d2h),
                     "what": "public API STSVerifyStep.step_host: H2D target+draft Q, draft capture, mask select, "
                             "sparse attention (one CUDA graph), D2H output"},
        "gpu_launches": int(launches),
        "launches_per_stage": stage_launches,
        "clocks": clocks.summary(),
        "wall_s_timed_loop": round(wall, 3),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# sequence-sharded path (config c4: 1M context, KV split by sequence over ranks)
# ---------------------------------------------------------------------------

def run_sharded(args, world, rank, local):
    import torch
    import torch.distributed as dist

    from paper_2605_15508_b200 import SparsityConfig, _lib, sharded
    from paper_2605_15508_b200.verify import algorithmic_bytes, config_shape, random_mapping_table

    local = 0 if args.one_gpu else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
        drive = lambda proto: sharded.run(proto)  # noqa: E731
    else:
        drive = sharded.run_single
    _lib.load()
    shape = config_shape(args.config, **shape_overrides(args))
    budget = round(1.0 - args.sparsity, 10)
    cfg = SparsityConfig(budget=budget, page_size=args.page_size)
    table = random_mapping_table(shape, seed=5)
    # heads x sequence: head group g = rank // sp holds kv-heads [g*Hkv/hp, ...),
    # the sp ranks of a group split the sequence and exchange among themselves
    hp = args.head_groups or (2 if args.config == "c5" and world % 2 == 0 and world > 1 else 1)
    if world % hp or shape.target_kv_heads % hp:
        raise SystemExit(f"--head-groups {hp} must divide the GPU count {world} and the kv-heads")
    sp = world // hp
    g, srank = rank // sp, rank % sp
    kv_bytes = (shape.batch * shape.target_layers * shape.target_kv_heads * shape.n_kv * shape.head_dim * 4
                + shape.batch * shape.draft_layers * shape.draft_kv_heads * shape.n_kv * shape.draft_head_dim * 2)
    if kv_bytes / world > 170e9:
        raise SystemExit(f"{args.config} needs {kv_bytes / 1e9:.0f} GB of KV cache: run it on >= "
                         f"{math.ceil(kv_bytes / 170e9)} GPUs (torchrun --nproc-per-node N bench.py --gpus N)")
    group = None
    if world > 1 and hp > 1:
        groups = [dist.new_group(list(range(h * sp, (h + 1) * sp))) for h in range(hp)]
        group = groups[g]
        drive = lambda proto: sharded.run(proto, group=group)  # noqa: E731
    step = sharded.ShardedVerifyStep(shape, cfg, table, srank, sp, device=dev, align=max(64, args.page_size),
                                     head_groups=hp, head_group=g)
    if args.merge == "p2p" and world > 1:
        step.enable_p2p(group)
    dq, dk, tq, tk, tv = sharded.local_synthetic_inputs(shape, step.bounds, srank, dev, seed=0, head_groups=hp,
                                                       head_group=g)
    dqv, dkv, q, k, v = step.local_views(dq, dk, tq, tk, tv, full=False)
    flush = L2Flush(dev, args.flush)
    st = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        drive(step.step(dqv, dkv, q, k, v))
        drive(step.attend_dense(q, k, v))
    barrier()
    assert step.status.item() == 0, f"device status {step.status.item()}"
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    t_cap, t_sel, t_att, t_den = [], [], [], []
    lib = _lib.load()
    launches0 = lib.sts_launch_count()  # our kernels launched inside the timed loop (library counter)
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            flush()
            barrier()
            e = [ev() for _ in range(3)]
            e[0].record(st)
            drive(step.capture(dqv, dkv))
            e[1].record(st)
            drive(step.build_masks())
            e[2].record(st)
            flush()
            barrier()
            e3, e4 = ev(), ev()
            e3.record(st)
            drive(step.attend(q, k, v))
            e4.record(st)
            flush()
            barrier()
            e5, e6 = ev(), ev()
            e5.record(st)
            drive(step.attend_dense(q, k, v))
            e6.record(st)
            torch.cuda.synchronize()
            t_cap.append(e[0].elapsed_time(e[1]) * 1e3)
            t_sel.append(e[1].elapsed_time(e[2]) * 1e3)
            t_att.append(e3.elapsed_time(e4) * 1e3)
            t_den.append(e5.elapsed_time(e6) * 1e3)
    launches = int(lib.sts_launch_count() - launches0)
    # end to end through the public API: host Q in, host O out (every rank)
    h_tq, h_dq = tq.cpu().pin_memory(), dq.cpu().pin_memory()
    h_out = torch.empty(step.out.shape, dtype=step.out.dtype).pin_memory()
    d_tq, d_dq = torch.empty_like(tq), torch.empty_like(dq)
    dqe, _, qe, _, _ = step.local_views(d_dq, dk, d_tq, tk, tv, full=False)
    t_e2e = []
    for i in range(args.warmup + args.steps):
        flush()
        barrier()
        e0, e1 = ev(), ev()
        e0.record(st)
        d_tq.copy_(h_tq, non_blocking=True)
        d_dq.copy_(h_dq, non_blocking=True)
        out, _ = drive(step.step(dqe, dkv, qe, k, v))
        h_out.copy_(out, non_blocking=True)
        e1.record(st)
        torch.cuda.synchronize()
        if i >= args.warmup:
            t_e2e.append(e0.elapsed_time(e1) * 1e3)

    mean = lambda x: float(sum(x) / len(x))  # noqa: E731
    stats = torch.tensor([mean(t_att), mean(t_den), mean(t_cap), mean(t_sel), mean(t_e2e)], device=dev)
    cnt_local = torch.tensor([float(step.cnt.float().sum().item())], device=dev)
    if world > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.MAX)
        dist.all_reduce(cnt_local, op=dist.ReduceOp.SUM)
    att, den, cap, sel, e2e = stats.tolist()
    keys_per_unit = cnt_local.item() / shape.target_units
    nbytes = algorithmic_bytes(shape, keys_per_unit)
    peak, peak_src = peaks()
    achieved = nbytes / (att * 1e-6) / 1e9 / world  # per GPU
    h2d = tq.numel() * tq.element_size() + dq.numel() * dq.element_size()
    d2h = step.out.numel() * step.out.element_size()
    rounds = step.selector.rounds
    line = {
        "metric": METRIC, "value": round(att, 2), "unit": "us", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(att / 1e3, 5), "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded N(0,1) bf16 Q/K/V per shard, random head mapping)",
        "config": {"workload": f"{args.config}: {MODEL_NAMES.get(args.config, 'synthetic')} shapes, {shape.context} "
                               f"context, KV sharded over {world} GPU(s) ({hp} head groups x {sp} sequence shards), "
                               f"batch {shape.batch}, gamma "
                               f"{shape.gamma}, sparsity {args.sparsity}, mode S, page_size {args.page_size}",
                   "context": shape.context, "batch": shape.batch, "gamma": shape.gamma, "mode": "S",
                   "page_size": args.page_size, "shard_positions": step.n_loc,
                   "keys_per_kv_head": round(keys_per_unit, 1), "l2": flush.describe(),
                   "parallelism": f"{hp} head group(s) x sequence-sharded x{sp} ({args.dist_backend} histogram allreduce + "
                                  f"{'peer-memory' if args.merge == 'p2p' and world > 1 else 'all-gather'} LSE merge)"},
        "dense_us": round(den, 2), "speedup_vs_dense": round(den / att, 3),
        "mask_build_us": {"draft_capture": round(cap, 2), "select": round(sel, 2)},
        "sts_step_us": round(cap + sel + att, 2), "step_speedup_vs_dense": round(den / (cap + sel + att), 3),
        "hbm_gbs_per_gpu": round(achieved, 1),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": None,
                     "kernel": "sts_sparse_decode + all-gather + sts_lse_merge (per GPU)",
                     "algorithmic_bytes_per_launch": int(nbytes / world), "peak_source": peak_src},
        "collectives_per_step": {"capture": 1, "select": rounds + 1, "attend": 2},
        "cpu_baseline": None,
        "e2e": {"value": round(e2e, 2), "unit": "us", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "what": "ShardedVerifyStep.step per rank: H2D target+draft Q, capture, select, attention, merge, D2H"},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
