"""Sequence-sharded (context-parallel) STS verify step — SURVEY §8(e).

For multi-million-token contexts the KV cache of every (layer, kv-head) is
split by sequence over P ranks: rank r holds the contiguous, page-aligned
positions ``[lo_r, hi_r)`` of the target K/V and of the draft K.  One verify
step then runs, on every rank, with only three kinds of exchange:

  capture   local draft LSE per row -> all-gather (P x rows floats) ->
            global LSE (sts_lse_merge, LSE only) -> local probability rows
  select    global top-k threshold by radix rounds over an all-reduced
            histogram (int32 [rows][2048] per round, every (layer, head) row at
            once) + one all-gather of per-rank tie counts, so the union of the
            ranks' selections is bit-exactly the single-GPU selection of the
            concatenated row (ties to the lowest GLOBAL index,
            src/numkit.py:84); sts_dist_select_* in include/sts_b200.h
  attend    local gathered flash-decode over the selected local keys ->
            fp32 partial (O_r, LSE_r) -> all-gather -> LSE merge (every rank
            ends with the full output)

The exchanges are written as a *protocol*: a generator that yields collective
requests.  ``run`` services them with torch.distributed (NCCL over NVLink on
the B200 box; gloo in the CPU tests), ``run_lockstep`` drives P virtual ranks
in one process (P shards of one GPU's tensors; the single-GPU tests use it to
check the full sharded path on real kernels).  Collective count per step is
O(radix rounds + 3), independent of layers and heads.

Mode S only (one key set per (layer, kv-head), scores reduced over the
gamma+1 rows and the GQA group): the mode the north star names.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _lib, kernels
from ._lib import call, ptr, stream_handle
from .kernels import Workspace
from .sparsity import SparsityConfig
from .verify_step import VerifyShape, _nvtx

ALL_REDUCE_SUM = "all_reduce_sum"
ALL_GATHER = "all_gather"
BARRIER = "barrier"  # device-side barrier over the ranks' symmetric-memory handle (p2p merge)


def shard_bounds(n: int, nranks: int, align: int = 1):
    """Contiguous, ``align``-aligned position ranges [lo, hi) per rank."""
    if nranks < 1:
        raise ValueError("nranks must be >= 1")
    per = -(-n // nranks)
    per = -(-per // align) * align
    return [(min(r * per, n), min((r + 1) * per, n)) for r in range(nranks)]


# ---------------------------------------------------------------------------
# collective drivers
# ---------------------------------------------------------------------------

def run(protocol, group=None):
    """Service one rank's protocol with torch.distributed collectives."""
    import torch.distributed as dist

    result = None
    try:
        req = next(protocol)
        while True:
            kind = req[0]
            if kind == ALL_REDUCE_SUM:
                dist.all_reduce(req[1], op=dist.ReduceOp.SUM, group=group)
            elif kind == BARRIER:
                req[1].barrier(channel=0)
            elif kind == ALL_GATHER:
                src, dst = req[1], req[2]
                if dist.get_backend(group) == "nccl":
                    dist.all_gather_into_tensor(dst, src, group=group)
                else:  # gloo (CPU tests): list form
                    P = dist.get_world_size(group)
                    dist.all_gather(list(dst.view(P, -1).unbind(0)), src.reshape(-1), group=group)
            else:  # pragma: no cover - protocol bug
                raise RuntimeError(f"unknown collective {kind!r}")
            req = protocol.send(None)
    except StopIteration as stop:
        result = stop.value
    return result


def run_single(protocol):
    """Service a one-rank protocol (P = 1): every collective is the identity."""
    result = None
    try:
        req = next(protocol)
        while True:
            if req[0] == ALL_GATHER:
                req[2].view(-1).copy_(req[1].view(-1))
            req = protocol.send(None)  # (all-reduce over one rank and barriers are no-ops)
    except StopIteration as stop:
        result = stop.value
    return result


def run_lockstep(protocols):
    """Drive P virtual ranks' protocols in one process, rank order = list
    order.  Every rank must issue the same sequence of collectives (they do:
    the protocol has no data-dependent control flow)."""
    P = len(protocols)
    results = [None] * P
    reqs = [next(p) for p in protocols]
    while True:
        kinds = {r[0] for r in reqs}
        if len(kinds) != 1:
            raise RuntimeError(f"ranks diverged: {kinds}")
        kind = reqs[0][0]
        if kind == ALL_REDUCE_SUM:
            tot = reqs[0][1].clone()
            for r in reqs[1:]:
                tot += r[1]
            for r in reqs:
                r[1].copy_(tot)
        elif kind == ALL_GATHER:
            stacked = torch.stack([r[1] for r in reqs]).view(-1)
            for r in reqs:
                r[2].view(-1).copy_(stacked)
        elif kind == BARRIER:
            pass  # virtual ranks share one stream: already ordered
        else:  # pragma: no cover
            raise RuntimeError(f"unknown collective {kind!r}")
        done = 0
        for i, p in enumerate(protocols):
            try:
                reqs[i] = p.send(None)
            except StopIteration as stop:
                results[i] = stop.value
                done += 1
        if done == P:
            return results
        if done:
            raise RuntimeError("ranks finished at different steps")


# ---------------------------------------------------------------------------
# distributed selection (one rank)
# ---------------------------------------------------------------------------

class DistSelector:
    """Buffers + protocol of the sharded top-k for ``rows`` logical rows whose
    local part holds ``n_local`` positions (include/sts_b200.h
    sts_dist_select_*)."""

    def __init__(self, rows: int, n_local: int, page_size: int, nranks: int, device):
        lib = _lib.load()
        self.rows, self.n_local, self.page_size, self.nranks = rows, n_local, page_size, nranks
        self.rounds = int(lib.sts_dist_select_rounds(page_size))
        self.ws = torch.empty(int(lib.sts_dist_select_workspace_bytes(rows, n_local, page_size)),
                              dtype=torch.uint8, device=device)
        self.hist_local = torch.zeros((rows, _lib.STS_DIST_BINS), dtype=torch.int32, device=device)
        self.hist_global = torch.zeros_like(self.hist_local) if nranks > 1 else self.hist_local
        self.ties_local = torch.zeros((rows,), dtype=torch.int32, device=device)
        self.ties_all = torch.zeros((nranks, rows), dtype=torch.int32, device=device)

    def protocol(self, scores: torch.Tensor, *, row_src, n_global: int, lo: int, k_top: int, rank: int,
                 include_current=False, include_sink=False, recent_window=0, tail_len=0, n_kv_local=None,
                 idx, cnt, status=None, stream=None):
        """Generator: yields the collective requests; fills idx/cnt (local offsets)."""
        if scores.dtype != torch.float32 or scores.stride(1) != 1:
            raise ValueError("scores must be row-major fp32")
        nsrc = row_src.shape[1] if row_src is not None else 1
        g = _lib.DistRows(ptr(scores), scores.stride(0), ptr(row_src), nsrc, self.rows, int(n_global), int(lo),
                          self.n_local, int(k_top), self.page_size)
        gp = C_ref(g)
        st = stream_handle(stream)
        wlen = self.ws.numel()
        call("sts_dist_select_begin", gp, ptr(self.hist_local), ptr(self.ws), wlen, st)
        for r in range(self.rounds):
            if self.nranks == 1:  # the global histogram IS the local one: no copy, no collective
                call("sts_dist_select_round", gp, r, ptr(self.hist_local), ptr(self.hist_local),
                     ptr(self.ties_local) if r == self.rounds - 1 else None, ptr(self.ws), wlen, st)
                continue
            self.hist_global.copy_(self.hist_local)
            yield (ALL_REDUCE_SUM, self.hist_global)
            last = r == self.rounds - 1
            call("sts_dist_select_round", gp, r, ptr(self.hist_global), ptr(self.hist_local),
                 ptr(self.ties_local) if last else None, ptr(self.ws), wlen, st)
        yield (ALL_GATHER, self.ties_local, self.ties_all)
        flags = (_lib.STS_SEL_CURRENT if include_current else 0) | (_lib.STS_SEL_SINK if include_sink else 0)
        n_kv_local = self.n_local if n_kv_local is None else int(n_kv_local)
        call("sts_dist_select_finish", gp, int(rank), self.nranks, ptr(self.ties_all), flags, int(recent_window),
             int(tail_len), n_kv_local, ptr(idx), idx.stride(0), ptr(cnt), ptr(status), ptr(self.ws), wlen, st)
        return idx, cnt


def C_ref(struct):
    """Address of a ctypes struct for a ``const T*`` argument (the struct
    object must outlive the call; callers keep it in their frame)."""
    import ctypes

    return ctypes.addressof(struct)


# ---------------------------------------------------------------------------
# sharded verify step (one rank)
# ---------------------------------------------------------------------------

class ShardedVerifyStep:
    """One rank of the sequence-sharded mode-S verify step.

    The rank holds positions [lo, hi) of the n_kv = context + gamma + 1 cached
    positions: target K/V views [U, hi-lo, d] and draft K [Ud, hi-lo, dd].
    Queries (target [U, M, d], draft [Ud, G*R, dd]) are replicated.
    """

    def __init__(self, shape: VerifyShape, sparsity: SparsityConfig, mapping_table, rank: int, nranks: int,
                 device=None, align: int | None = None, head_groups: int = 1, head_group: int = 0):
        """``rank`` / ``nranks``: position in the SEQUENCE group (the ranks
        whose collectives this step exchanges).  ``head_groups`` > 1 adds
        heads parallelism (BASELINE config 5): this rank holds only target
        kv-heads [head_group * Hkv / head_groups, ...) of every layer and batch
        (their K/V and queries), while the draft capture is computed for all
        draft heads (any of them can map onto this group's target heads)."""
        s = self.shape = shape
        self.cfg = sparsity
        self.rank, self.nranks = int(rank), int(nranks)
        if s.target_kv_heads % head_groups:
            raise ValueError("target kv-heads must divide evenly into head groups")
        self.head_groups, self.head_group = int(head_groups), int(head_group)
        self.hkv = s.target_kv_heads // head_groups
        self.kv_lo = head_group * self.hkv
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        R, base = s.rows, s.context
        align = sparsity.page_size if align is None else align
        if align % sparsity.page_size:
            raise ValueError("shard alignment must be a multiple of the page size")
        self.bounds = shard_bounds(s.n_kv, nranks, align)
        self.lo, self.hi = self.bounds[rank]
        self.n_loc = self.hi - self.lo
        table = np.asarray(mapping_table, dtype=np.int64)
        if table.shape != (s.target_layers, s.target_q_heads):
            raise ValueError(f"mapping table must be [{s.target_layers}, {s.target_q_heads}]")
        Gt = s.target_group
        nd = s.draft_layers * s.draft_q_heads
        self.budget = sparsity.tokens_for_context(base + 1)  # per round, src/specdec.py:331
        ps = sparsity.page_size
        self.k_top = self.budget if ps == 1 else -(-self.budget // ps)
        self.n_cols = max(4, -(-self.n_loc // 4) * 4)
        src = (np.arange(s.batch)[:, None, None, None] * nd
               + table.reshape(1, s.target_layers, s.target_kv_heads, Gt))
        src = src[:, :, self.kv_lo : self.kv_lo + self.hkv]  # this head group's kv-heads
        self.row_src = torch.from_numpy(np.ascontiguousarray(src).reshape(-1, Gt).astype(np.int32)).to(dev)
        self.U = U = s.batch * s.target_layers * self.hkv  # target units held here
        # draft side
        self.ws_draft = Workspace(dev)
        GRd = s.draft_group * R
        self.lse_local = torch.empty((s.draft_units, GRd), dtype=torch.float32, device=dev)
        self.lse_all = torch.empty((nranks, s.draft_units, GRd), dtype=torch.float32, device=dev)
        self.lse_global = torch.empty((s.draft_units * GRd,), dtype=torch.float32, device=dev)
        self.draft_rows = torch.zeros((s.batch * nd, self.n_cols), dtype=torch.float32, device=dev)
        # selection
        self.selector = DistSelector(U, self.n_loc, ps, nranks, dev)
        cap = min(self.n_loc, self.k_top * ps + int(sparsity.include_sink) + sparsity.recent_window + R)
        self.idx_ld = max(1, cap)
        self.idx = torch.empty((U, self.idx_ld), dtype=torch.int32, device=dev)
        self.cnt = torch.empty((U,), dtype=torch.int32, device=dev)
        # attention
        self.M = Gt * R
        self.ws_dec = Workspace(dev)
        self.o_part = torch.empty((U, self.M, s.head_dim), dtype=torch.float32, device=dev)
        self.l_part = torch.empty((U, self.M), dtype=torch.float32, device=dev)
        self.o_all = torch.empty((nranks, U, self.M, s.head_dim), dtype=torch.float32, device=dev)
        self.l_all = torch.empty((nranks, U, self.M), dtype=torch.float32, device=dev)
        self.out = torch.empty((U, self.M, s.head_dim), dtype=torch.bfloat16, device=dev)
        self.lse = torch.empty((U, self.M), dtype=torch.float32, device=dev)
        self.status = torch.zeros((1,), dtype=torch.int32, device=dev)

    # -- protocols (generators yielding collective requests) -----------------
    def capture(self, draft_q, draft_k, stream=None):
        s, R = self.shape, self.shape.rows
        G = s.draft_group
        with _nvtx("sts.capture"):
            kernels.draft_lse(draft_q, draft_k, G=G, R=R, base=s.context, n_keys=self.n_loc, pos_offset=self.lo,
                              out=self.lse_local, workspace=self.ws_draft, stream=stream)
        yield (ALL_GATHER, self.lse_local, self.lse_all)
        with _nvtx("sts.capture"):
            self._capture_probs(draft_q, draft_k, s, G, R, stream)

    def _capture_probs(self, draft_q, draft_k, s, G, R, stream):
        kernels.lse_merge(None, self.lse_all.view(self.nranks, -1), lse_out=self.lse_global, stream=stream)
        kernels.draft_probs(draft_q, draft_k, self.lse_global.view(s.draft_units, -1), G=G, R=R, base=s.context,
                            mode="S", n_keys=self.n_loc, pos_offset=self.lo, out=self.draft_rows, stream=stream)

    def build_masks(self, stream=None):
        s, cfg = self.shape, self.cfg
        yield from self.selector.protocol(
            self.draft_rows, row_src=self.row_src, n_global=s.context, lo=self.lo, k_top=self.k_top,
            rank=self.rank, include_current=False, include_sink=cfg.include_sink,
            recent_window=cfg.recent_window, tail_len=s.rows, n_kv_local=self.n_loc, idx=self.idx, cnt=self.cnt,
            status=self.status, stream=stream)

    # -- p2p merge: partials in symmetric memory, merged over peer pointers ----
    def enable_p2p(self, group=None):
        """Put this rank's partial (O, LSE) in torch symmetric memory and merge
        by reading every rank's buffer over NVLink in one kernel
        (sts_lse_merge_ptrs) after a device-side barrier, instead of an NCCL
        all-gather + local merge.  Needs torch.distributed initialised."""
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm

        grp = group or dist.group.WORLD
        try:
            symm.enable_symm_mem_for_group(grp.group_name)
        except Exception:  # pragma: no cover - already enabled / not needed
            pass
        U, M, d = self.out.shape
        buf = symm.empty(U * M * d + U * M, dtype=torch.float32, device=self.device)
        hdl = symm.rendezvous(buf, grp)
        self._use_part_buffer(buf, hdl.buffer_ptrs_dev, hdl)

    def _use_part_buffer(self, buf, ptrs_dev, hdl=None):
        U, M, d = self.out.shape
        self.part_buf = buf
        self.o_part = buf[: U * M * d].view(U, M, d)
        self.l_part = buf[U * M * d:].view(U, M)
        self.part_ptrs_dev = ptrs_dev  # int (device address) or a device int64 tensor of the P pointers
        self.p2p_handle = hdl
        self.merge_mode = "p2p"

    def _merge(self, stream=None):
        if getattr(self, "merge_mode", "gather") == "p2p":
            U, M, d = self.out.shape
            ptrs = self.part_ptrs_dev if isinstance(self.part_ptrs_dev, int) else self.part_ptrs_dev.data_ptr()
            yield (BARRIER, self.p2p_handle)  # every rank's partial is written and visible
            call("sts_lse_merge_ptrs", ptrs, self.nranks, U * M, d, 0, U * M * d, _lib.STS_DTYPE_BF16,
                 ptr(self.out), ptr(self.lse), stream_handle(stream))
            yield (BARRIER, self.p2p_handle)  # nobody rewrites its partial while peers still read it
            return
        yield (ALL_GATHER, self.o_part, self.o_all)
        yield (ALL_GATHER, self.l_part, self.l_all)
        U, M, d = self.out.shape
        kernels.lse_merge(self.o_all.view(self.nranks, U * M, d), self.l_all.view(self.nranks, U * M),
                          out_dtype=torch.bfloat16, out=self.out.view(U * M, d), lse_out=self.lse.view(-1),
                          stream=stream)

    def attend(self, target_q, target_k, target_v, stream=None):
        s = self.shape
        with _nvtx("sts.attend"):
            kernels.sparse_decode(target_q, target_k, target_v, idx=self.idx, cnt=self.cnt, causal_base=s.context,
                                  rows_per_head=s.rows, pos_offset=self.lo, out=self.o_part, lse=self.l_part,
                                  out_dtype=torch.float32, status=self.status, workspace=self.ws_dec,
                                  stream=stream)
        yield from self._merge(stream)
        return self.out, self.lse

    def attend_dense(self, target_q, target_k, target_v, stream=None):
        s = self.shape
        kernels.sparse_decode(target_q, target_k, target_v, n_dense=self.n_loc, causal_base=s.context,
                              rows_per_head=s.rows, pos_offset=self.lo, out=self.o_part, lse=self.l_part,
                              out_dtype=torch.float32, status=self.status, workspace=self.ws_dec, stream=stream)
        yield from self._merge(stream)
        return self.out, self.lse

    def step(self, draft_q, draft_k, target_q, target_k, target_v, stream=None):
        yield from self.capture(draft_q, draft_k, stream)
        yield from self.build_masks(stream)
        return (yield from self.attend(target_q, target_k, target_v, stream))

    # -- layouts -------------------------------------------------------------
    def local_views(self, dq, dk, tq, tk, tv, full: bool = True):
        """Unit views of this rank's inputs.  ``full``: dk/tk/tv hold all n_kv
        positions (single-process tests) and are sliced to [lo, hi); else they
        already are the local shard."""
        s = self.shape
        sl = slice(self.lo, self.hi) if full else slice(0, self.n_loc)
        Gt = s.target_group
        if tq.shape[2] == s.target_q_heads and self.head_groups > 1:  # full-head tensors: take this group
            tq = tq[:, :, self.kv_lo * Gt : (self.kv_lo + self.hkv) * Gt]
        if tk.shape[2] == s.target_kv_heads and self.head_groups > 1:
            tk = tk[:, :, self.kv_lo : self.kv_lo + self.hkv]
            tv = tv[:, :, self.kv_lo : self.kv_lo + self.hkv]
        q = tq.reshape(self.U, self.M, s.head_dim)
        k = tk.flatten(0, 2)[:, sl]
        v = tv.flatten(0, 2)[:, sl]
        dqv = dq.reshape(s.draft_units, s.draft_group * s.rows, s.draft_head_dim)
        dkv = dk.reshape(s.draft_units, dk.shape[-2], s.draft_head_dim)[:, sl]
        return dqv, dkv, q, k, v


def local_synthetic_inputs(shape: VerifyShape, bounds, rank: int, device, dtype=torch.bfloat16, seed: int = 0,
                           head_groups: int = 1, head_group: int = 0):
    """This rank's shard of synthetic_inputs (verify_step.py): the same seeded
    values a single GPU would hold at positions [lo, hi), generated shard by
    shard so no rank ever materialises the full cache (1M-token contexts)."""
    s = shape
    lo, hi = bounds[rank]
    n = hi - lo
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

    hkv = s.target_kv_heads // head_groups
    hq = hkv * s.target_group
    hs = 100000 * head_group  # head groups draw independent values
    tq = randn((s.batch, s.target_layers, hq, s.rows, s.head_dim), seed + 0 + hs)
    tk = randn((s.batch, s.target_layers, hkv, n, s.head_dim), seed + 1 + 1000 * rank + hs)
    tv = randn((s.batch, s.target_layers, hkv, n, s.head_dim), seed + 2 + 1000 * rank + hs)
    dq = randn((s.batch, s.draft_layers, s.draft_q_heads, s.rows, s.draft_head_dim), seed + 3)
    dk = randn((s.batch, s.draft_layers, s.draft_kv_heads, n, s.draft_head_dim), seed + 4 + 1000 * rank)
    return dq, dk, tq, tk, tv


def link_p2p_lockstep(steps):
    """Single-process stand-in for ``enable_p2p`` (virtual ranks on one GPU):
    each rank's partials go to its own buffer and the merge reads all of them
    through a device pointer array — the same kernel and addressing as the
    symmetric-memory path, without NVLink."""
    U, M, d = steps[0].out.shape
    bufs = [torch.empty(U * M * d + U * M, dtype=torch.float32, device=st.device) for st in steps]
    ptrs = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device=steps[0].device)
    for st, b in zip(steps, bufs):
        st._use_part_buffer(b, ptrs)
    return bufs, ptrs
