"""One STS verify step on the GPU: draft-score capture -> mask build -> sparse
target attention for the gamma+1 verification rows of every (batch, layer,
kv-head).

This is the device-resident form of the reference round
(src/specdec.py:324-352): ``propose`` records draft attention rows
(:150-167), ``_verification_masks`` turns them into per-target-head masks
(:219-233), ``verify`` runs the masked target block (:170-209) and the
correction decode adds the (gamma+1)-th row (:345-352).  Here all gamma+1
rows are stacked (the vLLM layout) and processed in four launches:

  1. sts_draft_lse    draft rows' log-sum-exp           (draft K read once)
  2. sts_draft_probs  p = exp(s - lse), reduced (mode S) or per row (mode R)
  3. sts_select_topk  radix top-k per target (layer, kv-head) [mode S] or per
                      draft row [mode R] (+ sts_row_union for GQA, mode R)
  4. sts_sparse_decode gathered flash-decode over the selected keys

Mode S (north-star design): one key set per (layer, kv-head),
scores summed over the gamma+1 rows and the GQA group's mapped draft heads;
every row also attends its own in-block causal prefix.  Mode R
(reference-exact): every (target head, row) keeps its own reference mask;
the kernel gathers the union per kv-head and applies per-row membership bits.

All buffers are allocated once in ``__init__``; ``step`` allocates nothing.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, kernels
from .kernels import Workspace
from .sparsity import SparsityConfig


def _nvtx(name):
    """NVTX push/pop range around a stage's launches (``ncu --nvtx
    --nvtx-include "sts.attend/"`` selects the stage; a no-op cost otherwise)."""
    return torch.cuda.nvtx.range(name)


@dataclass(frozen=True)
class VerifyShape:
    batch: int
    context: int          # committed positions (base); rows sit at base .. base+gamma
    gamma: int
    target_layers: int
    target_q_heads: int
    target_kv_heads: int
    head_dim: int
    draft_layers: int
    draft_q_heads: int
    draft_kv_heads: int
    draft_head_dim: int

    @property
    def rows(self) -> int:  # R = gamma + 1 stacked verification rows
        return self.gamma + 1

    @property
    def n_kv(self) -> int:  # positions in the cache during verify
        return self.context + self.rows

    @property
    def target_group(self) -> int:
        return self.target_q_heads // self.target_kv_heads

    @property
    def draft_group(self) -> int:
        return self.draft_q_heads // self.draft_kv_heads

    @property
    def target_units(self) -> int:
        return self.batch * self.target_layers * self.target_kv_heads

    @property
    def draft_units(self) -> int:
        return self.batch * self.draft_layers * self.draft_kv_heads


def random_mapping_table(shape: VerifyShape, seed: int = 0) -> np.ndarray:
    """Synthetic head mapping: target (layer, q-head) -> flattened draft q-head
    (draft_layer * draft_q_heads + draft_head), drawn uniformly (one-to-many,
    global search like src/headmap.py:83-125 would produce)."""
    rng = np.random.default_rng(seed)
    n_draft = shape.draft_layers * shape.draft_q_heads
    return rng.integers(0, n_draft, size=(shape.target_layers, shape.target_q_heads)).astype(np.int32)


class STSVerifyStep:
    """Preallocated GPU pipeline for one verify step (see module docstring)."""

    def __init__(self, shape: VerifyShape, sparsity: SparsityConfig, mapping_table, mode: str = "S",
                 device=None, schedule: int = 0, long_row_min=None):
        if mode not in ("S", "R"):
            raise ValueError("mode must be 'S' or 'R'")
        if shape.target_q_heads % shape.target_kv_heads or shape.draft_q_heads % shape.draft_kv_heads:
            raise ValueError("q heads must be a multiple of kv heads")
        self.shape = s = shape
        self.cfg = sparsity
        self.mode = mode
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        R, base = s.rows, s.context
        table = np.asarray(mapping_table, dtype=np.int64)
        if table.shape != (s.target_layers, s.target_q_heads):
            raise ValueError(f"mapping table must be [{s.target_layers}, {s.target_q_heads}]")
        Gt = s.target_group
        nd = s.draft_layers * s.draft_q_heads
        # per-round budget (src/specdec.py:331): b(base + 1)
        self.budget = sparsity.tokens_for_context(base + 1)
        self.n_draft_cols = -(-s.n_kv // 4) * 4
        self.ws_draft, self.ws_sel, self.ws_dec = Workspace(dev), Workspace(dev), Workspace(dev)

        # draft side
        self.draft_lse = torch.empty((s.draft_units, s.draft_group * R), dtype=torch.float32, device=dev)
        if mode == "S":
            self.draft_rows = torch.zeros((s.batch * nd, self.n_draft_cols), dtype=torch.float32, device=dev)
            # row_src[(b, l, g), hh] = b*nd + table[l, g*Gt + hh]
            src = (np.arange(s.batch)[:, None, None, None] * nd
                   + table.reshape(1, s.target_layers, s.target_kv_heads, Gt))
            self.row_src = torch.from_numpy(src.reshape(-1, Gt).astype(np.int32)).to(dev)
            self.idx_ld = kernels.index_capacity(base, self.budget, sparsity.page_size, False,
                                                 sparsity.include_sink, sparsity.recent_window, R)
            self.idx = torch.empty((s.target_units, self.idx_ld), dtype=torch.int32, device=dev)
            self.cnt = torch.empty((s.target_units,), dtype=torch.int32, device=dev)
            self.member = None
            # long rows (>= long_row_min committed positions, default 64K): the
            # chunk-parallel radix select of the sharded path at P = 1 (every
            # pass spread over (row, chunk) CTAs) instead of one CTA per row.
            # Measured (tools/select_route_ab.py): c3 token 973 -> 796 us, c3
            # page 16 1376 -> 1218 us; at c2 (32K) select_kernel stays faster
            # (token 63 vs 105 us, page 16 112 vs 177 us)
            lr_min = int(os.environ.get("STS_LONG_ROW", "65536")) if long_row_min is None else int(long_row_min)
            self._dist = None
            if base >= lr_min and s.target_units <= 65535:
                from .sharded import DistSelector

                self._dist = DistSelector(s.target_units, s.n_kv, sparsity.page_size, 1, dev)
                self._dist_k = self.budget if sparsity.page_size == 1 else -(-self.budget // sparsity.page_size)
        else:
            rows_total = s.batch * nd * R
            self.draft_rows = torch.zeros((rows_total, self.n_draft_cols), dtype=torch.float32, device=dev)
            self.row_len = torch.from_numpy(np.tile(base + 1 + np.arange(R, dtype=np.int32), s.batch * nd)).to(dev)
            self.sel_ld = kernels.index_capacity(s.n_kv, sparsity.budget, sparsity.page_size, True,
                                                 sparsity.include_sink, sparsity.recent_window, 0)
            self.sel_idx = torch.empty((rows_total, self.sel_ld), dtype=torch.int32, device=dev)
            self.sel_cnt = torch.empty((rows_total,), dtype=torch.int32, device=dev)
            # union lists: unit (b, l, g), row m = hh*R + i -> draft row ((b*nd + table)*R + i)
            dr = (np.arange(s.batch)[:, None, None, None] * nd
                  + table.reshape(1, s.target_layers, s.target_kv_heads, Gt))  # [B, L, Hkv, Gt]
            src = dr[..., None] * R + np.arange(R)  # [B, L, Hkv, Gt, R]
            self.union_src = torch.from_numpy(src.reshape(-1, Gt * R).astype(np.int32)).to(dev)
            self.idx_ld = s.n_kv
            self.bitmap = torch.empty((s.target_units, s.n_kv), dtype=torch.int32, device=dev)
            self.idx = self.cnt = self.member = None
        # target side
        M = Gt * R
        self.M = M
        self.out = torch.empty((s.target_units, M, s.head_dim), dtype=torch.bfloat16, device=dev)
        self.lse = torch.empty((s.target_units, M), dtype=torch.float32, device=dev)
        self.status = torch.zeros((1,), dtype=torch.int32, device=dev)
        # attention work schedule (kernels.sparse_decode): 0 = auto; tests force
        # stream-K (1) or cluster sizes 2..8 to cover every instance
        self.schedule = int(schedule)
        # unit groups of the host-buffer attention pipeline (see attend_host)
        # (2 measured best at c2: 157 vs 200 µs for 1, 200 for 3 — tools/gpu_e2e_chunks.sh)
        self.host_chunks = int(os.environ.get("STS_HOST_CHUNKS", "2"))
        # host-buffer attention: K/V bytes pulled into L2 while Q is copied in
        self.l2_prefetch_bytes = 32 << 20  # 24-48 MB: 134 vs 140 us at c2 (tools/e2e_direct_probe.py)

    # -- the four stages ----------------------------------------------------------
    def capture(self, draft_q, draft_k, stream=None):
        """Stages 1-2: draft log-sum-exp and probability rows (score capture)."""
        s, R = self.shape, self.shape.rows
        with _nvtx("sts.capture"):
            self._capture(draft_q, draft_k, s, R, stream)

    def _capture(self, draft_q, draft_k, s, R, stream):
        kernels.draft_lse(draft_q, draft_k, G=s.draft_group, R=R, base=s.context, n_keys=s.n_kv,
                          out=self.draft_lse, workspace=self.ws_draft, stream=stream)
        kernels.draft_probs(draft_q, draft_k, self.draft_lse, G=s.draft_group, R=R, base=s.context,
                            mode=self.mode, n_keys=s.n_kv, out=self.draft_rows, stream=stream)

    def build_masks(self, stream=None):
        """Stage 3: radix top-k selection (+ union for mode R)."""
        with _nvtx("sts.select"):
            self._build_masks(stream)

    def _build_masks(self, stream):
        s, cfg = self.shape, self.cfg
        if self.mode == "S" and self._dist is not None:
            from .sharded import run_single

            run_single(self._dist.protocol(
                self.draft_rows, row_src=self.row_src, n_global=s.context, lo=0, k_top=self._dist_k, rank=0,
                include_current=False, include_sink=cfg.include_sink, recent_window=cfg.recent_window,
                tail_len=s.rows, n_kv_local=s.n_kv, idx=self.idx, cnt=self.cnt, status=self.status, stream=stream))
        elif self.mode == "S":
            kernels.select_topk(self.draft_rows, row_src=self.row_src, n_common=s.context,
                                budget=int(self.budget), page_size=cfg.page_size, include_current=False,
                                include_sink=cfg.include_sink, recent_window=cfg.recent_window,
                                tail_len=s.rows, out=self.idx, cnt=self.cnt, status=self.status,
                                workspace=self.ws_sel, stream=stream)
        else:
            kernels.select_topk(self.draft_rows, row_len=self.row_len, budget=cfg.budget,
                                page_size=cfg.page_size, include_current=True, include_sink=cfg.include_sink,
                                recent_window=cfg.recent_window, out=self.sel_idx, cnt=self.sel_cnt,
                                status=self.status, workspace=self.ws_sel, stream=stream)
            self.idx, self.member, self.cnt = kernels.row_union(
                self.sel_idx, self.sel_cnt, self.union_src, M=self.M, n_max=s.n_kv, bitmap=self.bitmap,
                status=self.status, stream=stream)

    def attend(self, target_q, target_k, target_v, stream=None):
        """Stage 4: gathered sparse flash-decode of the stacked rows."""
        s = self.shape
        causal = s.context if self.mode == "S" else -1
        with _nvtx("sts.attend"):
            return kernels.sparse_decode(target_q, target_k, target_v, idx=self.idx, cnt=self.cnt,
                                         member=self.member, causal_base=causal, rows_per_head=s.rows,
                                         schedule=self.schedule, out=self.out, lse=self.lse, status=self.status,
                                         workspace=self.ws_dec, stream=stream)

    def attend_dense(self, target_q, target_k, target_v, out=None, lse=None, stream=None):
        """Dense baseline on the same kernel: every cached key, causal tail."""
        s = self.shape
        with _nvtx("sts.dense"):
            return kernels.sparse_decode(target_q, target_k, target_v, n_dense=s.n_kv, causal_base=s.context,
                                         rows_per_head=s.rows,
                                         out=out if out is not None else self.out,
                                         lse=lse if lse is not None else self.lse, status=self.status,
                                         workspace=self.ws_dec, stream=stream)

    def step(self, draft_q, draft_k, target_q, target_k, target_v, stream=None):
        self.capture(draft_q, draft_k, stream)
        self.build_masks(stream)
        return self.attend(target_q, target_k, target_v, stream)

    # -- host-buffer API (queries in from pinned host memory, output back out) --
    _GRAPH_CACHE = 32

    def _graph(self, key, fn, keep=()):
        """CUDA graph of ``fn`` (captured once per key; replays launch no Python).
        ``keep``: host tensors the graph reads or writes by address (the key
        holds their pointers): held as long as the graph, so no other tensor
        can take their memory while a replay may still touch it."""
        if not hasattr(self, "_graphs"):
            self._graphs = {}
        ent = self._graphs.get(key)
        if ent is None:
            if len(self._graphs) >= self._GRAPH_CACHE:
                # bounded: callers passing fresh host buffers every call would
                # otherwise grow the cache (and the buffers it holds) forever;
                # evict the oldest once no replay of it can still be running
                torch.cuda.synchronize(self.device)
                self._graphs.pop(next(iter(self._graphs)))
            fn()  # warm-up outside capture (workspace allocations happen here)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                fn()
            ent = self._graphs[key] = (g, tuple(t for t in keep if t is not None))
        return ent[0]

    def _host_buffers(self, h_dq, h_tq):
        """Device staging buffers for host queries (allocated once per shape)."""
        if getattr(self, "_d_tq", None) is None or self._d_tq.shape != h_tq.shape:
            self._d_tq = torch.empty(h_tq.shape, dtype=h_tq.dtype, device=self.device)
        if h_dq is not None and (getattr(self, "_d_dq", None) is None or self._d_dq.shape != h_dq.shape):
            self._d_dq = torch.empty(h_dq.shape, dtype=h_dq.dtype, device=self.device)
        return getattr(self, "_d_dq", None), self._d_tq

    def attend_host(self, h_tq, target_k, target_v, h_out, chunks=None, direct_out=None):
        """Target attention with host queries: H2D copy of Q [B, L, Hq, R, d]
        (pinned), the attention, D2H copy of the output into ``h_out`` (pinned,
        shaped like ``self.out``).  The masks are the ones the last
        ``build_masks`` produced.

        ``direct_out`` (default: when ``h_out`` is pinned and contiguous): the attention
        kernel writes the output straight into ``h_out`` over the host link
        (pinned memory is device-mapped), so no D2H copy trails the kernel and
        the result is bit-identical to the device-resident ``attend`` (one
        launch).  Measured at c2: 138-142 µs vs 149-152 µs for the best
        copy-engine form (``tools/e2e_direct_probe.py``).

        Otherwise ``chunks`` > 1 pipelines the copies with the kernel: the units
        are cut into ``chunks`` contiguous groups and, inside one CUDA graph,
        the H2D of group c+1 and the D2H of group c-1 run on side streams while
        group c attends, so the link time hides behind the HBM-bound kernel.
        """
        direct_out, h_dst = self._direct_view(h_out, direct_out)
        if direct_out:
            chunks = 1 if chunks is None else int(chunks)
        else:
            chunks = self.host_chunks if chunks is None else int(chunks)
        _, d_tq = self._host_buffers(None, h_tq)
        q, k, v = self.target_views(d_tq, target_k, target_v)
        idx_ptr = self.idx.data_ptr() if self.idx is not None else 0
        if direct_out:
            key = ("attend_host_direct", chunks, self.l2_prefetch_bytes, h_tq.data_ptr(), h_out.data_ptr(),
                   target_k.data_ptr(), target_v.data_ptr(), idx_ptr)
            self._graph(key, lambda: self._attend_pipelined(h_tq, d_tq, q, k, v, h_dst, max(1, chunks),
                                                            direct_out=True), keep=(h_tq, h_out)).replay()
            return h_out
        if chunks <= 1:
            d_tq.copy_(h_tq, non_blocking=True)
            key = ("attend", target_k.data_ptr(), target_v.data_ptr(), idx_ptr)
            self._graph(key, lambda: self.attend(q, k, v)).replay()
            h_out.copy_(self.out, non_blocking=True)
            return h_out
        key = ("attend_host", chunks, self.l2_prefetch_bytes, h_tq.data_ptr(), h_out.data_ptr(), target_k.data_ptr(),
               target_v.data_ptr(), idx_ptr)
        self._graph(key, lambda: self._attend_pipelined(h_tq, d_tq, q, k, v, h_out, chunks),
                    keep=(h_tq, h_out)).replay()
        return h_out

    def _prefetch_first_rows(self, k, v, u0, u1, stream):
        """While the first queries cross the host link: the K/V rows each CTA
        of the attention reads first, into L2 (``l2_prefetch_bytes`` in all;
        0 disables). The shares follow the schedule the decode will use."""
        if not self.l2_prefetch_bytes or self.idx is None:
            return
        s = self.shape
        nu = u1 - u0
        sched = int(_lib.load().sts_sparse_decode_schedule(nu, self.M, s.head_dim, self.idx_ld, self.schedule))
        parts = sched if sched >= 2 else 1
        row = 2 * s.head_dim * k.element_size()  # K and V
        kpp = int(self.l2_prefetch_bytes // (nu * parts * row))
        if kpp > 0:
            kernels.kv_prefetch_l2(k, v, idx=self.idx[u0:u1], cnt=self.cnt[u0:u1], parts=parts, keys_per_part=kpp,
                                   stream=stream)

    def _direct_view(self, h_out, direct_out):
        """Whether the kernel writes ``h_out`` itself, and ``h_out`` viewed as
        ``step.out`` for that: by default when h_out is pinned, contiguous and
        holds step.out's elements in its dtype; ``direct_out=True`` requires it."""
        ok = (h_out.is_pinned() and h_out.is_contiguous() and h_out.numel() == self.out.numel()
              and h_out.dtype == self.out.dtype)
        if direct_out is None:
            direct_out = ok
        elif direct_out and not ok:
            raise ValueError("direct_out needs a pinned, contiguous h_out with step.out's size and dtype")
        return bool(direct_out), (h_out.view(self.out.shape) if direct_out else h_out)

    def _attend_pipelined(self, h_tq, d_tq, q, k, v, h_out, chunks, direct_out=False):
        s = self.shape
        U = s.target_units
        C = max(1, min(chunks, U))
        main = torch.cuda.current_stream(self.device)
        s_in, s_out = self._streams()
        dq_ = d_tq.view(U, -1)
        hq = h_tq.view(U, -1) if h_tq is not None else None  # None: the queries are on the device already
        ho = h_out.view(U, -1)
        s_in.wait_stream(main)
        s_out.wait_stream(main)
        causal = s.context if self.mode == "S" else -1
        for c in range(C):
            u0, u1 = U * c // C, U * (c + 1) // C
            if hq is not None:
                with torch.cuda.stream(s_in):
                    dq_[u0:u1].copy_(hq[u0:u1], non_blocking=True)
                if c == 0:
                    self._prefetch_first_rows(k[u0:u1], v[u0:u1], u0, u1, main)
                main.wait_stream(s_in)
            member = self.member[u0:u1] if self.member is not None else None
            kernels.sparse_decode(q[u0:u1], k[u0:u1], v[u0:u1], idx=self.idx[u0:u1], cnt=self.cnt[u0:u1],
                                  member=member, causal_base=causal, rows_per_head=s.rows, schedule=self.schedule,
                                  out=h_out[u0:u1] if direct_out else self.out[u0:u1], lse=self.lse[u0:u1],
                                  status=self.status, workspace=self.ws_dec, stream=main)
            if direct_out:
                continue
            s_out.wait_stream(main)
            with torch.cuda.stream(s_out):
                ho[u0:u1].copy_(self.out[u0:u1].view(u1 - u0, -1), non_blocking=True)
        main.wait_stream(s_out)

    def step_host(self, h_dq, draft_k, h_tq, target_k, target_v, h_out, chunks=None, direct_out=None):
        """The whole verify step with host queries (draft Q [B, Ld, Hqd, R, dd]
        and target Q), replayed as one CUDA graph; output copied to ``h_out``.

        With ``chunks`` > 1 (default ``host_chunks``) the copies ride inside the
        graph: the target-Q H2D runs on a side stream under the capture and
        select stages, and the output D2H of each unit group overlaps the
        attention of the next.  With a pinned ``h_out`` the attention writes the
        output there directly (see ``attend_host``)."""
        direct_out, h_dst = self._direct_view(h_out, direct_out)
        chunks = 1 if direct_out else (self.host_chunks if chunks is None else int(chunks))
        d_dq, d_tq = self._host_buffers(h_dq, h_tq)
        dq, dk = self.draft_views(d_dq, draft_k)
        q, k, v = self.target_views(d_tq, target_k, target_v)
        if chunks <= 1 and not direct_out:
            d_dq.copy_(h_dq, non_blocking=True)
            d_tq.copy_(h_tq, non_blocking=True)
            key = ("step", draft_k.data_ptr(), target_k.data_ptr(), target_v.data_ptr())
            self._graph(key, lambda: self.step(dq, dk, q, k, v)).replay()
            h_out.copy_(self.out, non_blocking=True)
            return h_out

        def body():
            main = torch.cuda.current_stream(self.device)
            s_in, _ = self._streams()
            s_in.wait_stream(main)
            with torch.cuda.stream(s_in):
                d_dq.copy_(h_dq, non_blocking=True)
            main.wait_stream(s_in)
            with torch.cuda.stream(s_in):  # under capture + select
                d_tq.copy_(h_tq, non_blocking=True)
            self.capture(dq, dk)
            self.build_masks()
            main.wait_stream(s_in)
            self._attend_pipelined(None, d_tq, q, k, v, h_dst, chunks, direct_out=direct_out)

        key = ("step_host", chunks, direct_out, h_dq.data_ptr(), h_tq.data_ptr(), h_out.data_ptr(), draft_k.data_ptr(),
               target_k.data_ptr(), target_v.data_ptr())
        self._graph(key, body, keep=(h_dq, h_tq, h_out)).replay()
        return h_out

    def _streams(self):
        if getattr(self, "_copy_streams", None) is None:
            self._copy_streams = (torch.cuda.Stream(device=self.device), torch.cuda.Stream(device=self.device))
        return self._copy_streams

    # -- layouts ------------------------------------------------------------------
    def target_views(self, q, k, v):
        """[B, L, Hq, R, d] q and [B, L, Hkv, N, d] caches -> kernel unit views."""
        s = self.shape
        U = s.target_units
        def units(x):  # keep the row stride (interleaved K|V views are not contiguous)
            return x.flatten(0, 2) if x.dim() == 5 else x
        return q.reshape(U, self.M, s.head_dim), units(k), units(v)

    def draft_views(self, q, k):
        s = self.shape
        U = s.draft_units
        return q.reshape(U, s.draft_group * s.rows, s.draft_head_dim), k.reshape(U, k.shape[-2], s.draft_head_dim)


def synthetic_inputs(shape: VerifyShape, device, dtype=torch.bfloat16, seed: int = 0, n_max=None,
                     layout: str = "separate"):
    """Seeded synthetic inputs: Q, K, V ~ N(0,1); draft q/K too.

    Returns draft_q [B, Ld, Hqd, R, dd], draft_k [B, Ld, Hkvd, N, dd],
    target_q [B, L, Hq, R, d], target_k/v [B, L, Hkv, N, d]; N = n_kv.
    layout "interleaved" stores the target cache as [B, L, Hkv, N, 2, d]
    (K|V of one token adjacent) and returns k/v as strided views of it.
    Generated in chunks on the device to bound peak memory.
    """
    s = shape
    n = s.n_kv if n_max is None else n_max
    g = torch.Generator(device=device)

    def randn(shape_, seed_):
        g.manual_seed(seed_)
        t = torch.empty(shape_, dtype=dtype, device=device)
        flat = t.view(-1)
        step = 1 << 28
        for i in range(0, flat.numel(), step):
            m = min(step, flat.numel() - i)
            flat[i : i + m] = torch.randn(m, generator=g, device=device, dtype=torch.float32).to(dtype)
        return t

    tq = randn((s.batch, s.target_layers, s.target_q_heads, s.rows, s.head_dim), seed + 0)
    if layout == "interleaved":
        kv = randn((s.batch, s.target_layers, s.target_kv_heads, n, 2, s.head_dim), seed + 1)
        tk, tv = kv[..., 0, :], kv[..., 1, :]
    else:
        tk = randn((s.batch, s.target_layers, s.target_kv_heads, n, s.head_dim), seed + 1)
        tv = randn((s.batch, s.target_layers, s.target_kv_heads, n, s.head_dim), seed + 2)
    dq = randn((s.batch, s.draft_layers, s.draft_q_heads, s.rows, s.draft_head_dim), seed + 3)
    dk = randn((s.batch, s.draft_layers, s.draft_kv_heads, n, s.draft_head_dim), seed + 4)
    return dq, dk, tq, tk, tv


# BASELINE.json configs (SURVEY §8a model shapes)
CONFIGS = {
    "c1": dict(batch=1, context=4096, gamma=4, target_layers=4, target_q_heads=8, target_kv_heads=8, head_dim=64,
               draft_layers=2, draft_q_heads=4, draft_kv_heads=4, draft_head_dim=64),
    "c2": dict(batch=1, context=32768, gamma=4, target_layers=32, target_q_heads=32, target_kv_heads=8,
               head_dim=128, draft_layers=16, draft_q_heads=32, draft_kv_heads=8, draft_head_dim=64),
    "c3": dict(batch=8, context=131072, gamma=4, target_layers=28, target_q_heads=28, target_kv_heads=4,
               head_dim=128, draft_layers=24, draft_q_heads=14, draft_kv_heads=2, draft_head_dim=64),
    "c4": dict(batch=1, context=1048576, gamma=4, target_layers=32, target_q_heads=32, target_kv_heads=8,
               head_dim=128, draft_layers=16, draft_q_heads=32, draft_kv_heads=8, draft_head_dim=64),
    "c5": dict(batch=4, context=262144, gamma=4, target_layers=80, target_q_heads=64, target_kv_heads=8,
               head_dim=128, draft_layers=16, draft_q_heads=32, draft_kv_heads=8, draft_head_dim=64),
}


def config_shape(name: str, **overrides) -> VerifyShape:
    d = dict(CONFIGS[name])
    d.update(overrides)
    return VerifyShape(**d)


def algorithmic_bytes(shape: VerifyShape, keys_per_unit: float, e: int = 2, dense: bool = False) -> float:
    """bytes = U*|S|*d*2*e (K,V) + U*|S|*4 (idx) + 2*B*L*Hq*R*d*e (Q,O)
    + B*L*Hq*R*4 (LSE)."""
    s = shape
    U = s.target_units
    kv = U * keys_per_unit * s.head_dim * 2 * e
    idx = 0 if dense else U * keys_per_unit * 4
    rows = s.batch * s.target_layers * s.target_q_heads * s.rows
    return kv + idx + 2 * rows * s.head_dim * e + rows * 4
