#!/usr/bin/env python
"""STS verify-step benchmark on B200 (driver contract: one JSON line on rank 0).

Metric (BASELINE.json): target-attention µs per verify step at 90% sparsity,
with speedup vs a dense decode on the same GPU and achieved HBM GB/s.

  python bench.py [--gpus N] [--steps 20] [--warmup 5] [--config c2] [--mode S]
  python bench.py --impl reference ...   # the reference CPU path (specsparse, baseline/_ref)

Workloads.  N = 1: BASELINE config 2 — Llama-3.2-1B draft -> Llama-3.1-8B
target shapes, 32K context, batch 1, 90% sparsity, gamma = 4 (5 stacked rows
x GQA 4), synthetic N(0,1) bf16 Q/K/V, random head mapping.  N > 1: config 4
— the 8B target at 1M context with the KV cache sharded by sequence over the
N GPUs (strong scaling: the same workload at every N); the line also carries
the one-GPU time of that same workload measured on rank 0's GPU after the
sharded run, so the curve is self-contained.  ``--gpus N`` without a
launcher (no WORLD_SIZE) spawns the N ranks itself through
torch.distributed.run.

A "step" is one verify step: draft-score capture, mask build, sparse target
attention over all layers x kv-heads.  ``value`` is the sparse target-attention
time of the step (inputs resident in HBM, L2 flushed before every timed stage);
capture / select, the dense decode, the end-to-end public-API time (host->device
Q copies and the device->host output copy inside the timed region) and an
oracle parity check of sampled units (after the timed loop, on the timed
run's own outputs) are reported beside it.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import platform
import socket
import subprocess
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
REF_DIR = ROOT / "baseline" / "_ref"


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
    ap.add_argument("--schedule", type=int, default=0, help="attention work schedule (0 auto, 1 stream-K, C clusters)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="bound of the CPU baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the c2 mode-R and fp32 side measurements")
    ap.add_argument("--parity-units", type=int, default=32, help="units checked against the oracle after timing")
    ap.add_argument("--eager", action="store_true", help="time stages as eager launches instead of CUDA graphs")
    ap.add_argument("--graph-collectives", action="store_true",
                    help="N > 1: capture each sharded stage, NCCL collectives included, in a CUDA graph")
    ap.add_argument("--flush", default="clean", choices=["clean", "write", "none"], help="L2 flush between stages")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="collective backend for N > 1 (gloo + --one-gpu: functional check on a single GPU)")
    ap.add_argument("--one-gpu", action="store_true", help="map every rank to cuda:0 (functional checks only)")
    ap.add_argument("--head-groups", type=int, default=0,
                    help="heads x sequence sharding: ranks per head group = gpus / head_groups (0: 2 for c5, else 1)")
    ap.add_argument("--merge", default="gather", choices=["gather", "p2p"],
                    help="sharded path: NCCL all-gather + merge, or one peer-memory merge kernel over symmetric memory")
    ap.add_argument("--no-single-ref", action="store_true",
                    help="N > 1: skip the one-GPU time of the same workload on rank 0")
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


def workload_key(config, mode, page_size, layout, world, sparsity=0.9):
    return f"{config}:{mode}:s{sparsity:g}:ps{page_size}:{layout}:P{world}"


def ncu_traffic(key):
    """Per-launch DRAM bytes (ncu dram__bytes_read.sum + dram__bytes_write.sum)
    of the attention kernel for this workload, from the committed per-config
    ncu summaries (profiles/ncu_traffic.json, written by tools/ncu_traffic.py
    from `ncu --set full` captures of this bench); None if not captured."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None, None
    try:
        d = json.loads(p.read_text()).get(key)
    except Exception:
        return None, None
    if not d:
        return None, None
    return d.get("dram_bytes"), d.get("source")


def gather_floor(config, mode, sparsity):
    """The measured pure-gather floor of this workload's selection (K and V
    rows of every selected key, no math; tools/gather_probe.py), from the
    committed probe runs; None if not measured."""
    if mode != "S":
        return None
    for f in sorted((ROOT / "profiles").glob("r*/**/gather_probe*.json"), reverse=True):
        try:
            for line in f.read_text().splitlines():
                if not line.startswith("{"):
                    continue
                d = json.loads(line)
                w = d.get("workload", "")
                if w.split()[0] == config and abs(float(w.split()[-1].rstrip("%")) / (100 if w.endswith("%") else 1)
                                                  - sparsity) < 1e-6:
                    best = min(v for k, v in d.items() if k.startswith("gather_us"))
                    return {"us": best, "source": f"tools/gather_probe.py ({f.relative_to(ROOT)})"}
        except Exception:
            continue
    return None


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


def mean(x):
    return float(sum(x) / len(x))


# ---------------------------------------------------------------------------
# CPU reference path: the reference's own functions (specsparse installed in
# baseline/_ref) when present, else the oracle port of them
# ---------------------------------------------------------------------------

def _ref_impl():
    """('reference', sparsity, specdec, headmap) from baseline/_ref, or
    ('port', oracle module, None, None)."""
    if (REF_DIR / "specsparse").is_dir():
        if str(REF_DIR) not in sys.path:
            sys.path.insert(0, str(REF_DIR))
        import specsparse.headmap as H
        import specsparse.sparsity as S
        import specsparse.specdec as D

        return "reference", S, D, H
    from oracle import sts_oracle as O

    return "port", O, None, None


_KV_CACHE = {}


def _attn_call_worker(args):
    """One reference sparse_attention call (src/sparsity.py:152-173) on
    synthetic K/V (generated once per worker process and shape: the reference
    still converts the whole K/V to fp64 inside every call, :167-168); dense
    when k >= n (mask = arange(n))."""
    import numpy as np

    seed, n, d, k = args
    kind, S, _, _ = _ref_impl()
    rng = np.random.default_rng(seed)
    q = rng.standard_normal(d).astype(np.float32)
    if (n, d) not in _KV_CACHE:
        _KV_CACHE.clear()
        g = np.random.default_rng(n * 131 + d)
        _KV_CACHE[(n, d)] = (g.standard_normal((n, d)).astype(np.float32), g.standard_normal((n, d)).astype(np.float32))
    keys, vals = _KV_CACHE[(n, d)]
    mask = np.arange(n) if k >= n else np.sort(rng.choice(n, size=k, replace=False))
    t0 = time.perf_counter()
    S.sparse_attention(q, keys, vals, mask)
    return time.perf_counter() - t0


def _mask_build_worker(args):
    """One reference _verification_masks call (src/specdec.py:219-233) over
    ``heads`` draft heads x gamma rows + the correction row's
    remap_masks(draft_masks_decode(...)) (src/specdec.py:345-352), every target
    head mapped onto those draft heads; returns (seconds, draft heads)."""
    import numpy as np

    seed, base, gamma, heads, targets_per = args
    kind, S, D, H = _ref_impl()
    rng = np.random.default_rng(seed)

    def row(n):
        z = 2.0 * rng.standard_normal(n)
        w = np.exp(z - z.max())
        return (w / w.sum()).astype(np.float32)

    dheads = [(0, h) for h in range(heads)]
    rows = [{hd: row(base + i + 1) for hd in dheads} for i in range(gamma)]
    corr = {hd: row(base + gamma + 1) for hd in dheads}
    entries = {(t // (targets_per * heads), t % (targets_per * heads)): (dheads[t % heads], 0)
               for t in range(targets_per * heads)}
    if kind == "reference":
        cfg = S.SparsityConfig(budget=0.1)
        mapping = H.HeadMapping(k=cfg.tokens_for_context(base + 1), entries=entries, trace_set_id="bench",
                                draft_config=None, target_config=None)
        t0 = time.perf_counter()
        D._verification_masks(rows, base, cfg, mapping)
        S.remap_masks(S.draft_masks_decode(corr, cfg), mapping)
    else:
        cfg = S.OracleSparsityConfig(0.1)
        t0 = time.perf_counter()
        S.verification_masks(rows, base, cfg, entries)
        S.remap_masks(S.draft_masks_decode(corr, cfg), entries)
    return time.perf_counter() - t0


def _pool_time(fn, make_args, budget_s, workers):
    """Run fn (which returns the seconds of its timed reference call) over
    make_args(i) on `workers` concurrent processes for ~budget_s; return
    (effective seconds per call at that parallelism = mean call time / workers,
    calls).  Calls run concurrently, so memory-bandwidth contention between
    the processes is part of the measured call times."""
    import multiprocessing as mp

    t_end = time.perf_counter() + budget_s
    done, i = 0, 0
    if workers > 1:
        ctx = mp.get_context("fork")
        times = []
        with ctx.Pool(workers) as pool:
            while time.perf_counter() < t_end or done == 0:
                times.extend(pool.map(fn, [make_args(i + j) for j in range(workers)], chunksize=1))
                i += workers
                done += workers
        return sum(times) / len(times) / workers, done
    tot = 0.0
    while time.perf_counter() < t_end or done == 0:
        tot += fn(make_args(i))
        i += 1
        done += 1
    return tot / done, done


def host_info(workers):
    import numpy as np

    cpu = platform.processor() or ""
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                cpu = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    blas = None
    try:
        cfg = np.show_config(mode="dicts")
        b = cfg.get("Build Dependencies", {}).get("blas", {})
        blas = f"{b.get('name')} {b.get('version')}"
    except Exception:
        pass
    return {"cpu_model": cpu, "cpu_count": os.cpu_count(), "threads_used": workers,
            "OMP_NUM_THREADS": os.environ.get("OMP_NUM_THREADS"), "numpy": np.__version__, "blas": blas,
            "python": platform.python_version()}


def cpu_reference(shape, k_sel, budget_s, workers, items=("attention", "mask_build", "dense")):
    """The reference's CPU path timed on this host, each item
    on a bounded sample scaled linearly to one verify step:
      attention   sparse_attention per (layer, q-head, row): B*L*Hq*(gamma+1) calls
      mask_build  _verification_masks + correction remap over all draft heads
                  (sampled heads, scaled by draft heads / sampled heads)
      dense       the attention loop with mask = arange(n)
    Returns a dict of µs per step plus the sampling description."""
    kind, _, _, _ = _ref_impl()
    n, d = shape.n_kv, shape.head_dim
    calls = shape.batch * shape.target_layers * shape.target_q_heads * shape.rows
    per_item = budget_s / len(items)
    res = {"kind": kind, "calls_per_step": calls}
    # each call holds K/V fp32 + the reference's fp64 copies (src/sparsity.py:167-168): ~24 B per element
    w_attn = max(1, min(workers, int(8e9 // (24 * n * d))))
    if "attention" in items:
        per, done = _pool_time(_attn_call_worker, lambda i: (i, n, d, k_sel), per_item, w_attn)
        res["attention_us"] = per * calls * 1e6
        res["attention_sample"] = f"{done} sparse_attention calls (n={n}, d={d}, |S|={k_sel}) on {w_attn} processes"
    if "dense" in items:
        per, done = _pool_time(_attn_call_worker, lambda i: (10**6 + i, n, d, n), per_item, w_attn)
        res["dense_us"] = per * calls * 1e6
        res["dense_sample"] = f"{done} dense sparse_attention(arange(n)) calls on {w_attn} processes"
    if "mask_build" in items:
        heads = 2
        nd = shape.batch * shape.draft_layers * shape.draft_q_heads
        tp = max(1, (shape.batch * shape.target_layers * shape.target_q_heads) // nd)
        w_mask = max(1, min(workers, 16))
        per, done = _pool_time(_mask_build_worker, lambda i: (i, shape.context, shape.gamma, heads, tp), per_item,
                               w_mask)
        res["mask_build_us"] = per * (nd / heads) * 1e6
        res["mask_build_sample"] = (f"{done} _verification_masks(+correction) calls over {heads} draft heads x "
                                    f"{shape.gamma} rows of {shape.context} positions on {w_mask} processes, "
                                    f"scaled x{nd / heads:.0f} to all {nd} draft heads")
    return res


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2605_15508_b200.verify_step import config_shape

    shape = config_shape(args.config, **shape_overrides(args))
    budget = round(1.0 - args.sparsity, 10)
    k_sel = max(1, math.ceil(budget * (shape.context + 1))) + shape.rows
    workers = os.cpu_count() or 1
    vals = []
    per_step = max(1.0, args.cpu_seconds / max(args.steps, 1))
    r = None
    for i in range(args.warmup + args.steps):
        r = cpu_reference(shape, k_sel, per_step, workers, items=("attention",))
        if i >= args.warmup:
            vals.append(r["attention_us"])
    value = mean(vals)
    kind = r["kind"]
    sample = (("specsparse.sparsity.sparse_attention (the reference itself, baseline/_ref)" if kind == "reference"
               else "oracle sparse_attention (numpy restatement of src/sparsity.py:152-173)")
              + f": {r['attention_sample']} per step-sample, scaled to {r['calls_per_step']} calls/step "
                f"(extrapolated: a full c2+ verify step takes minutes on the CPU)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 1), "unit": "us",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(value / 1e3, 3),
        "higher_is_better": False, "scaling": "weak" if args.gpus == 1 else "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: target attention of one verify step (CPU reference path), "
                               f"{MODEL_NAMES.get(args.config)} shapes, {shape.context} context, batch {shape.batch}",
                   "sparsity": args.sparsity, "gamma": shape.gamma},
        "cpu_baseline": {"value": round(value, 1), "unit": "us", "cores": workers, "kind": kind, "sample": sample,
                         "host": host_info(workers)},
        "e2e": {"value": round(value, 1), "unit": "us", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------------------
# launcher (--gpus N without torchrun)
# ---------------------------------------------------------------------------

def spawn(args):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


# ---------------------------------------------------------------------------
# GPU path, one GPU (c2 by default)
# ---------------------------------------------------------------------------

def graph_of(fn, eager=False):
    import torch

    if eager:
        return fn
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g.replay


def run_single_gpu(args):
    import torch

    from oracle import parity
    from paper_2605_15508_b200 import SparsityConfig, _lib
    from paper_2605_15508_b200.verify_step import (STSVerifyStep, algorithmic_bytes, config_shape, random_mapping_table,
                                              synthetic_inputs)

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    lib = _lib.load()
    shape = config_shape(args.config, **shape_overrides(args))
    budget = round(1.0 - args.sparsity, 10)
    cfg = SparsityConfig(budget=budget, page_size=args.page_size)
    table = random_mapping_table(shape, seed=5)
    step = STSVerifyStep(shape, cfg, table, mode=args.mode, device=dev, schedule=args.schedule)
    dq, dk, tq, tk, tv = synthetic_inputs(shape, dev, seed=0, layout=args.layout)
    q, k, v = step.target_views(tq, tk, tv)
    dqv, dkv = step.draft_views(dq, dk)
    dense_out = torch.empty_like(step.out)
    dense_lse = torch.empty_like(step.lse)
    flush = L2Flush(dev, args.flush)
    st = torch.cuda.current_stream()

    for _ in range(args.warmup):
        step.step(dqv, dkv, q, k, v)
        step.attend_dense(q, k, v, out=dense_out, lse=dense_lse)
    torch.cuda.synchronize()
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
    for name, fn in stages.items():
        c0 = lib.sts_launch_count()
        if args.eager:
            fn()
        run_stage[name] = graph_of(fn, args.eager)
        stage_launches[name] = int(lib.sts_launch_count() - c0)  # our kernels per replay
    for _ in range(2):
        for fn in run_stage.values():
            fn()
    torch.cuda.synchronize()
    t = {name: [] for name in stages}
    with ClockSampler(0) as clocks:
        torch.cuda.synchronize()
        wall0 = time.perf_counter()
        for _ in range(args.steps):
            for name in ("capture", "select", "attend", "dense"):
                if name != "select":  # select reads the rows capture just wrote (L2-warm, as in a real step)
                    flush()
                e0, e1 = ev(), ev()
                e0.record(st)
                run_stage[name]()
                e1.record(st)
                t[name].append((e0, e1))
            torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
    us = {name: mean([a.elapsed_time(b) * 1e3 for a, b in pairs]) for name, pairs in t.items()}
    att, den, cap, sel = us["attend"], us["dense"], us["capture"], us["select"]

    # parity of the timed run's own outputs (graph replays) on sampled units
    par = None
    if args.mode == "S" and args.parity_units > 0:
        run_stage["capture"]()
        run_stage["select"]()
        run_stage["attend"]()
        torch.cuda.synchronize()
        units = parity.sample_units(shape.batch, shape.target_layers, shape.target_kv_heads, args.parity_units)
        par = parity.check_units(step, q, k, v, step.out, units)
        # the device masks vs masks from fp64 reference draft rows
        par["mask_agreement"] = parity.mask_agreement(step, dq, dk, units[:8])

    # end to end through the public API with host buffers (pinned), copies inside
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
    e2e, e2e_step = mean(t_e2e), mean(t_e2e_step)

    cnt = step.cnt.float().mean().item()
    nbytes = algorithmic_bytes(shape, cnt)
    dense_bytes = algorithmic_bytes(shape, shape.n_kv, dense=True)
    peak, peak_src = peaks()
    achieved = nbytes / (att * 1e-6) / 1e9
    key = workload_key(args.config, args.mode, args.page_size, args.layout, 1, args.sparsity)
    traffic, traffic_src = ncu_traffic(key)
    sched = int(lib.sts_sparse_decode_schedule(shape.target_units, step.M, shape.head_dim, step.idx_ld,
                                               args.schedule))
    launches = args.steps * sum(stage_launches.values())  # counted by the library (sts_launch_count)

    extras = {}
    if args.config == "c2" and args.mode == "S" and not args.no_extras:
        extras = side_measurements(args, shape, cfg, table, dq, dk, tq, tk, tv, flush, dev)

    cpu = None
    if not args.no_cpu_baseline:
        r = cpu_reference(shape, int(round(cnt)), args.cpu_seconds, os.cpu_count() or 1)
        cpu = {"value": round(r["attention_us"], 1), "unit": "us", "cores": os.cpu_count() or 1, "kind": r["kind"],
               "sample": r["attention_sample"] + f", scaled to {r['calls_per_step']} calls/step",
               "items_us_per_step": {"sparse_attention": round(r["attention_us"], 1),
                                     "mask_build": round(r["mask_build_us"], 1),
                                     "dense_attention": round(r["dense_us"], 1)},
               "items_sample": {"mask_build": r["mask_build_sample"], "dense_attention": r["dense_sample"]},
               "host": host_info(os.cpu_count() or 1)}

    h2d = tq.numel() * tq.element_size()
    h2d_step = h2d + dq.numel() * dq.element_size()
    d2h = step.out.numel() * step.out.element_size()
    line = {
        "metric": METRIC, "value": round(att, 2), "unit": "us", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(att / 1e3, 5), "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded N(0,1) bf16 Q/K/V, random head mapping)",
        "config": {"workload": f"{args.config}: {MODEL_NAMES.get(args.config, 'synthetic')} shapes, "
                               f"{shape.context} context, batch {shape.batch}, gamma {shape.gamma}, "
                               f"sparsity {args.sparsity}, mode {args.mode}, page_size {args.page_size}, "
                               f"kv layout {args.layout}",
                   "context": shape.context, "batch": shape.batch, "gamma": shape.gamma, "mode": args.mode,
                   "page_size": args.page_size, "kv_layout": args.layout,
                   "keys_per_kv_head": round(cnt, 1), "l2": flush.describe(),
                   "launch": "eager" if args.eager else "CUDA graph per stage",
                   "attention_schedule": "stream-K" if sched == 1 else f"{sched}-CTA clusters per unit",
                   "parallelism": "single"},
        "dense_us": round(den, 2), "speedup_vs_dense": round(den / att, 3),
        "mask_build_us": {"draft_capture": round(cap, 2), "select": round(sel, 2)},
        "sts_step_us": round(cap + sel + att, 2), "step_speedup_vs_dense": round(den / (cap + sel + att), 3),
        "hbm_gbs": round(achieved, 1), "dense_hbm_gbs": round(dense_bytes / (den * 1e-6) / 1e9, 1),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic, "traffic_source": traffic_src,
                     "kernel": "sts_sparse_decode: verify_decode_kernel (gathered flash-decode, cluster/DSMEM or "
                               "stream-K + piece merge)",
                     "algorithmic_bytes_per_launch": int(nbytes), "peak_source": peak_src,
                     **({"gather_floor_us": gf["us"], "frac_of_gather_floor": round(gf["us"] / att, 4),
                         "gather_floor_source": gf["source"]} if (gf := gather_floor(args.config, args.mode,
                                                                                     args.sparsity)) else {})},
        "parity": par,
        "cpu_baseline": cpu,
        "e2e": {"value": round(e2e, 2), "unit": "us", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "what": "public API STSVerifyStep.attend_host: H2D of the target Q from pinned host memory, sparse "
                        "target attention writing its output straight into the pinned host buffer (device-mapped; "
                        "the output crosses the host link inside the kernel); one CUDA graph",
                "output": "direct"},
        "e2e_step": {"value": round(e2e_step, 2), "unit": "us", "h2d_bytes_per_step": int(h2d_step),
                     "d2h_bytes_per_step": int(d2h),
                     "what": "public API STSVerifyStep.step_host: H2D target+draft Q (target Q under capture + "
                             "select), draft capture, mask select, sparse attention writing the pinned host output "
                             "(one CUDA graph)"},
        "gpu_launches": int(launches),
        "launches_per_stage": stage_launches,
        "clocks": clocks.summary(),
        "wall_s_timed_loop": round(wall, 3),
    }
    line.update(extras)
    print(json.dumps(line), flush=True)


def side_measurements(args, shape, cfg, table, dq, dk, tq, tk, tv, flush, dev):
    """c2 side lines: mode R (reference-exact per-row masks: union per kv-head
    + row-membership bits) with its union/k overfetch, and the fp32 CUDA-core
    parity kernel on the mode-S key lists."""
    import torch

    from paper_2605_15508_b200 import kernels
    from paper_2605_15508_b200.verify_step import STSVerifyStep

    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    st = torch.cuda.current_stream()

    def timed(fn, n):
        fn()
        g = graph_of(fn)
        g()
        torch.cuda.synchronize()
        out = []
        for _ in range(n):
            flush()
            e0, e1 = ev(), ev()
            e0.record(st)
            g()
            e1.record(st)
            torch.cuda.synchronize()
            out.append(e0.elapsed_time(e1) * 1e3)
        return mean(out)

    n = max(3, min(args.steps, 10))
    res = {}
    r = STSVerifyStep(shape, cfg, table, mode="R", device=dev)
    q, k, v = r.target_views(tq, tk, tv)
    dqv, dkv = r.draft_views(dq, dk)
    r.step(dqv, dkv, q, k, v)
    torch.cuda.synchronize()
    cap = timed(lambda: r.capture(dqv, dkv), n)
    sel = timed(lambda: r.build_masks(), n)
    att = timed(lambda: r.attend(q, k, v), n)
    union = r.cnt.float().mean().item()
    per_row = r.sel_cnt.float().mean().item()
    res["mode_r"] = {"attend_us": round(att, 2), "draft_capture_us": round(cap, 2), "select_us": round(sel, 2),
                     "keys_per_kv_head_union": round(union, 1), "keys_per_row_mask": round(per_row, 1),
                     "union_over_k": round(union / per_row, 3),
                     "what": "reference-exact per-(head,row) masks (specdec._verification_masks semantics); the "
                             "kernel gathers each kv-head's union of its 20 row masks and applies per-row membership "
                             "bits; synthetic draft rows are independent random draws, so the union nearly covers "
                             "the context"}
    del r
    # fp32 parity kernel (CUDA cores) on the same mode-S key lists
    s = STSVerifyStep(shape, cfg, table, mode="S", device=dev)
    q, k, v = s.target_views(tq, tk, tv)
    s.step(*s.draft_views(dq, dk), q, k, v)
    qf, kf, vf = q.float(), k.float(), v.float()
    outf = torch.empty(qf.shape, dtype=torch.float32, device=dev)
    lsef = torch.empty(qf.shape[:2], dtype=torch.float32, device=dev)
    att32 = timed(lambda: kernels.sparse_decode(qf, kf, vf, idx=s.idx, cnt=s.cnt, causal_base=shape.context,
                                                rows_per_head=shape.rows, splits=1, out=outf, lse=lsef), n)
    res["fp32_attend_us"] = round(att32, 2)
    del s, qf, kf, vf
    torch.cuda.empty_cache()
    return res


# ---------------------------------------------------------------------------
# sequence-sharded path (config c4: 1M context, KV split by sequence over ranks)
# ---------------------------------------------------------------------------

def measure_sharded(args, world, rank, local, group_world=None):
    """Time the sequence-sharded verify step on this rank (world == 1: the
    one-GPU point of the same workload).  Returns a dict of per-rank numbers."""
    import torch
    import torch.distributed as dist

    from paper_2605_15508_b200 import SparsityConfig, _lib, sharded
    from paper_2605_15508_b200.verify_step import config_shape, random_mapping_table

    dev = torch.device("cuda", local)
    lib = _lib.load()
    if world > 1:
        drive = lambda proto: sharded.run(proto)  # noqa: E731
    else:
        drive = sharded.run_single
    shape = config_shape(args.config, **shape_overrides(args))
    budget = round(1.0 - args.sparsity, 10)
    cfg = SparsityConfig(budget=budget, page_size=args.page_size)
    table = random_mapping_table(shape, seed=5)
    hp = args.head_groups or (2 if args.config == "c5" and world % 2 == 0 and world > 1 else 1)
    if world % hp or shape.target_kv_heads % hp:
        raise SystemExit(f"--head-groups {hp} must divide the GPU count {world} and the kv-heads")
    sp = world // hp
    g, srank = rank // sp, rank % sp
    kv_bytes = (shape.batch * shape.target_layers * shape.target_kv_heads * shape.n_kv * shape.head_dim * 4
                + shape.batch * shape.draft_layers * shape.draft_kv_heads * shape.n_kv * shape.draft_head_dim * 2)
    if kv_bytes / world > 170e9:
        raise SystemExit(f"{args.config} needs {kv_bytes / 1e9:.0f} GB of KV cache: run it on >= "
                         f"{math.ceil(kv_bytes / 170e9)} GPUs (python bench.py --gpus N)")
    if world > 1 and hp > 1:
        groups = [dist.new_group(list(range(h * sp, (h + 1) * sp))) for h in range(hp)]
        group = groups[g]
        drive = lambda proto: sharded.run(proto, group=group)  # noqa: E731
    else:
        group = None
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
    stages = {"capture": lambda: drive(step.capture(dqv, dkv)), "select": lambda: drive(step.build_masks()),
              "attend": lambda: drive(step.attend(q, k, v)), "dense": lambda: drive(step.attend_dense(q, k, v))}
    # one GPU: a CUDA graph per stage.  Several ranks: eager launches unless
    # --graph-collectives (NCCL collectives inside graph capture are not
    # exercised in this environment's single-GPU runs; a capture failing on
    # one rank only would hang the others, so it is opt-in)
    launch_mode = "eager"
    run_stage = dict(stages)
    if not args.eager and (world == 1 or args.graph_collectives):
        try:
            graphs = {name: graph_of(fn) for name, fn in stages.items()}
            for fn in graphs.values():
                fn()
            barrier()
            run_stage, launch_mode = graphs, "CUDA graph per stage (collectives captured)"
        except Exception as exc:  # pragma: no cover - depends on the backend
            launch_mode = f"eager (graph capture failed: {type(exc).__name__})"
            barrier()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    t = {name: [] for name in stages}
    launches0 = lib.sts_launch_count()
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            for name in ("capture", "select", "attend", "dense"):
                if name != "select":
                    flush()
                barrier()
                e0, e1 = ev(), ev()
                e0.record(st)
                run_stage[name]()
                e1.record(st)
                torch.cuda.synchronize()
                t[name].append(e0.elapsed_time(e1) * 1e3)
    launches = int(lib.sts_launch_count() - launches0)
    if launch_mode.startswith("CUDA graph"):
        # graph replays launch nothing through the library: count one eager step's launches per stage
        c0 = lib.sts_launch_count()
        for fn in stages.values():
            fn()
        launches = int(lib.sts_launch_count() - c0) * args.steps
    barrier()
    # the timed run's outputs: one more replay of the step, then parity
    run_stage["capture"]()
    run_stage["select"]()
    run_stage["attend"]()
    barrier()
    par = sharded_parity(args, step, q, k, v, world, rank, hp)
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
    res = {"attend": mean(t["attend"]), "dense": mean(t["dense"]), "capture": mean(t["capture"]),
           "select": mean(t["select"]), "e2e": mean(t_e2e), "cnt_sum": float(step.cnt.float().sum().item()),
           "launches": launches, "launch_mode": launch_mode, "clocks": clocks.summary(), "parity": par,
           "hp": hp, "sp": sp, "n_loc": step.n_loc, "rounds": step.selector.rounds, "shape": shape,
           "h2d": tq.numel() * tq.element_size() + dq.numel() * dq.element_size(),
           "d2h": step.out.numel() * step.out.element_size(), "l2": flush.describe()}
    del step, dq, dk, tq, tk, tv, dqv, dkv, q, k, v, h_tq, h_dq, h_out, d_tq, d_dq, flush
    return res


def sharded_parity(args, step, q, k, v, world, rank, hp):
    """Oracle parity of sampled units of the sharded step.  Every rank sends
    its local share (the units' local draft rows over its committed positions,
    its selected global positions and their K/V rows) to rank 0, which rebuilds
    the full rows and checks masks bit-exactly and the merged output within
    the bf16 tolerance."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from oracle import parity
    from oracle import sts_oracle as O

    if args.parity_units <= 0 or hp != 1:
        return None
    s = step.shape
    units = parity.sample_units(s.batch, s.target_layers, s.target_kv_heads, min(args.parity_units, 8), seed=3)
    cl = max(0, min(step.hi, s.context) - step.lo)  # committed positions held here
    share = []
    for u in units:
        src = step.row_src[u].long()
        rows = step.draft_rows.index_select(0, src)[:, :cl].cpu().numpy()
        c = int(step.cnt[u])
        loc = step.idx[u, :c].long()
        share.append((rows, (loc + step.lo).cpu().numpy(), k[u].index_select(0, loc).cpu(),
                      v[u].index_select(0, loc).cpu()))
    if world > 1:
        gathered = [None] * world if rank == 0 else None
        dist.gather_object(share, gathered, dst=0)
    else:
        gathered = [share]
    if rank != 0:
        return None
    cfg = parity.oracle_config(step.cfg)
    bad, max_err = [], 0.0
    for j, u in enumerate(units):
        parts = [g[j] for g in gathered]
        rows = np.concatenate([p[0] for p in parts], axis=1)
        got = np.concatenate([p[1] for p in parts]).astype(np.int64)
        want = O.mode_s_index_list(O.reduce_rows_fp32(list(rows)), s.context, s.rows, cfg)
        if not np.array_equal(got, want):
            bad.append(u)
            continue
        ks = torch.cat([p[2] for p in parts]).float().numpy()
        vs = torch.cat([p[3] for p in parts]).float().numpy()
        ref, _ = O.block_attention_rows(q[u].float().cpu().numpy(), ks, vs, got, causal_base=s.context,
                                        rows_per_head=s.rows)
        max_err = max(max_err, float(np.abs(step.out[u].float().cpu().numpy() - ref).max()))
    return {"units": len(units), "masks_bit_exact": not bad, "mask_mismatch_units": bad[:8],
            "max_abs_err": round(max_err, 6), "tol": parity.BF16_TOL, "attention_ok": max_err <= parity.BF16_TOL,
            "how": "ranks' shares gathered to rank 0; full rows rebuilt in rank order"}


def run_sharded(args, world, rank, local):
    import datetime

    import torch
    import torch.distributed as dist

    from paper_2605_15508_b200.verify_step import algorithmic_bytes

    local = 0 if args.one_gpu else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        timeout = datetime.timedelta(minutes=30)  # rank 0 measures the one-GPU point while the others wait
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev, timeout=timeout)
        else:
            dist.init_process_group("gloo", timeout=timeout)
    r = measure_sharded(args, world, rank, local)
    stats = torch.tensor([r["attend"], r["dense"], r["capture"], r["select"], r["e2e"]], device=dev)
    cnt_local = torch.tensor([r["cnt_sum"]], device=dev)
    if world > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.MAX)
        dist.all_reduce(cnt_local, op=dist.ReduceOp.SUM)
    att, den, cap, sel, e2e = stats.tolist()
    shape = r["shape"]
    import gc

    gc.collect()
    torch.cuda.empty_cache()
    single = None
    if world > 1 and not args.no_single_ref and not args.one_gpu and r["hp"] == 1:
        # the same workload on one GPU (rank 0's), measured after the sharded run
        if dist.get_backend() == "nccl":
            dist.barrier(device_ids=[local])
        else:
            dist.barrier()
        if rank == 0:
            one = measure_sharded(args, 1, 0, local)
            single = {"attend_us": round(one["attend"], 2), "dense_us": round(one["dense"], 2),
                      "capture_us": round(one["capture"], 2), "select_us": round(one["select"], 2),
                      "parity": one["parity"], "what": "the same c4 workload on one GPU (rank 0's), P = 1"}
            del one
            gc.collect()
            torch.cuda.empty_cache()
        dist.barrier()
    keys_per_unit = cnt_local.item() / shape.target_units
    nbytes = algorithmic_bytes(shape, keys_per_unit)
    peak, peak_src = peaks()
    achieved = nbytes / (att * 1e-6) / 1e9 / world  # per GPU
    key = workload_key(args.config, "S", args.page_size, "separate", world, args.sparsity)
    traffic, traffic_src = ncu_traffic(key)
    hp, sp = r["hp"], r["sp"]
    line = {
        "metric": METRIC, "value": round(att, 2), "unit": "us", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(att / 1e3, 5), "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded N(0,1) bf16 Q/K/V per shard, random head mapping)",
        "config": {"workload": f"{args.config}: {MODEL_NAMES.get(args.config, 'synthetic')} shapes, {shape.context} "
                               f"context, batch {shape.batch}, gamma {shape.gamma}, sparsity {args.sparsity}, mode S, "
                               f"page_size {args.page_size}, KV sharded by sequence over the GPUs",
                   "context": shape.context, "batch": shape.batch, "gamma": shape.gamma, "mode": "S",
                   "page_size": args.page_size, "shard_positions": r["n_loc"],
                   "keys_per_kv_head": round(keys_per_unit, 1), "l2": r["l2"], "launch": r["launch_mode"],
                   "parallelism": f"{hp} head group(s) x sequence-sharded x{sp} ({args.dist_backend} histogram "
                                  f"allreduce + {'peer-memory' if args.merge == 'p2p' and world > 1 else 'all-gather'}"
                                  f" LSE merge)"},
        "dense_us": round(den, 2), "speedup_vs_dense": round(den / att, 3),
        "mask_build_us": {"draft_capture": round(cap, 2), "select": round(sel, 2)},
        "sts_step_us": round(cap + sel + att, 2), "step_speedup_vs_dense": round(den / (cap + sel + att), 3),
        "hbm_gbs_per_gpu": round(achieved, 1),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic, "traffic_source": traffic_src,
                     "kernel": "sts_sparse_decode + all-gather + sts_lse_merge (per GPU)",
                     "algorithmic_bytes_per_launch": int(nbytes / world), "peak_source": peak_src},
        "collectives_per_step": {"capture": 1, "select": (r["rounds"] + 1) if sp > 1 else 0,
                                 "attend": 2 if sp > 1 else 0},
        "parity": r["parity"],
        "single_gpu": single,
        "cpu_baseline": None,
        "e2e": {"value": round(e2e, 2), "unit": "us", "h2d_bytes_per_step": int(r["h2d"]),
                "d2h_bytes_per_step": int(r["d2h"]),
                "what": "ShardedVerifyStep.step per rank: H2D target+draft Q, capture, select, attention, merge, D2H"},
        "gpu_launches": r["launches"],
        "clocks": r["clocks"],
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.config == "auto":
        args.config = "c2" if max(world, args.gpus) == 1 else "c4"
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn(args))
    if args.config in ("c4", "c5") or world > 1:
        return run_sharded(args, world, rank, local)
    return run_single_gpu(args)


if __name__ == "__main__":
    main()
