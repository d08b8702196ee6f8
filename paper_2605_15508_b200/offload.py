"""KV offload tier driven by the masks.

The target K/V stay in pinned host memory; per verify step the pages the
masks select are brought into an HBM page pool and the gathered decode runs
on the pool.  The three strategies of the reference's offload model
(src/offloadsim.py:153-211):

* ``full``      — K/V resident in HBM (``STSVerifyStep.attend``);
* ``on_demand`` — layer by layer: copy the layer's pages, then attend it
                  (transfers and compute serialised, nothing persists);
* ``prefetch``  — the masks are known before target layer 0 (STS's "know in
                  advance"): every layer's pages are queued on a copy stream
                  up front and layer l attends as soon as its pages landed,
                  so the host-link transfers overlap the attention of the
                  layers already resident.

Pages are ``position // page_size`` (the pages_touched wire format of
src/specdec.py:236-255); with page-granular selection (``SparsityConfig(
page_size=P)``) a step moves only the selected pages.  The in-block tail
keeps fixed pool ranks so the decode's causal test holds unchanged
(include/sts_b200.h sts_page_plan).
"""

from __future__ import annotations

import torch

from . import kernels
from ._lib import call, ptr, stream_handle


class PagedKVOffload:
    """Host-resident K/V of one ``STSVerifyStep`` (mode S) plus its HBM page pool."""

    def __init__(self, step, host_k: torch.Tensor, host_v: torch.Tensor, page_size: int = 16, copy_ctas: int = 32,
                 resident: bool = False, capacity_pages: int | None = None):
        s = step.shape
        if step.mode != "S":
            raise ValueError("the offload tier serves mode S key lists")
        if not (host_k.is_pinned() and host_v.is_pinned()):
            raise ValueError("host K/V must be pinned (page-locked) host tensors")
        if host_k.shape != host_v.shape or host_k.dim() != 3 or host_k.stride(-1) != 1:
            raise ValueError("host K/V must be [units, n_kv, d] with unit inner stride")
        self.step, self.s = step, s
        self.hk, self.hv = host_k, host_v
        self.P = int(page_size)
        self.copy_ctas = int(copy_ctas)
        dev = step.device
        U, n, d = host_k.shape
        self.U, self.n, self.d = U, n, d
        base = s.context
        self.tail_page0 = base // self.P
        last_page = (n - 1) // self.P
        ntail = last_page - self.tail_page0 + 1
        committed_pages = min(step.idx_ld, -(-base // self.P))
        if resident:
            # the fast tier's committed capacity per unit (the reference's
            # fast_tier_capacity, split per unit); default: twice the pages a
            # page-granular step selects
            if capacity_pages is None:
                capacity_pages = 2 * (-(-int(step.budget) // self.P) + 2)
            committed_pages = max(1, min(committed_pages, int(capacity_pages)))
        self.pages_ld = committed_pages + ntail
        self.tail_rank0 = self.pages_ld - ntail
        # tail rows sit at position - shift in the pool
        self.shift = (self.tail_page0 - self.tail_rank0) * self.P
        rows = self.pages_ld * self.P
        self.pool_k = torch.empty((U, rows, d), dtype=host_k.dtype, device=dev)
        self.pool_v = torch.empty((U, rows, d), dtype=host_k.dtype, device=dev)
        self.pages = torch.empty((U, self.pages_ld), dtype=torch.int32, device=dev)
        self.npages = torch.empty((U,), dtype=torch.int32, device=dev)
        self.idx_pool = torch.empty_like(step.idx)
        self.copy_stream = torch.cuda.Stream(device=dev)
        # resident=True: the pool keeps pages across steps with LRU eviction
        # (the reference's "prefetch" strategy, src/offloadsim.py:173-209) and
        # a step copies only its missing pages; capacity = capacity_pages slots
        self.resident = bool(resident)
        self.step_no = 0
        if self.resident:
            self.slot_page = torch.full((U, self.pages_ld), -1, dtype=torch.int32, device=dev)
            self.slot_last = torch.full((U, self.pages_ld), -1, dtype=torch.int32, device=dev)
            self.slots = torch.empty((U, self.pages_ld), dtype=torch.int32, device=dev)
        # unit groups = (batch, layer): the attention runs group by group
        self.group = s.target_kv_heads
        self.groups = U // self.group

    def plan(self, stream=None):
        """Pages of this step's masks and the key lists in pool rows (one
        launch).  Resident pool: only the pages not already held, and their
        slots (LRU eviction)."""
        st = self.step
        if self.resident:
            call("sts_page_cache_plan", ptr(st.idx), st.idx.stride(0), ptr(st.cnt), self.U, self.P, self.tail_page0,
                 self.tail_rank0, ptr(self.slot_page), ptr(self.slot_last), self.pages_ld, self.tail_rank0,
                 self.step_no, ptr(self.pages), ptr(self.slots), ptr(self.npages), ptr(self.idx_pool),
                 ptr(st.status), stream_handle(stream))
            self.step_no += 1
            return
        call("sts_page_plan", ptr(st.idx), st.idx.stride(0), ptr(st.cnt), self.U, self.P, self.tail_page0,
             self.tail_rank0, ptr(self.pages), self.pages_ld, ptr(self.npages), ptr(self.idx_pool), ptr(st.status),
             stream_handle(stream))

    def _copy(self, g0: int, g1: int, stream=None):
        hk = self.hk
        call("sts_page_copy", ptr(hk), ptr(self.hv), hk.stride(0), hk.stride(1), self.n, ptr(self.pool_k),
             ptr(self.pool_v), self.pool_k.stride(0), self.d, hk.element_size(), ptr(self.pages), self.pages_ld,
             ptr(self.npages), ptr(self.slots) if self.resident else None, g0 * self.group, g1 * self.group, self.P,
             self.tail_page0, self.tail_rank0, self.copy_ctas, stream_handle(stream))

    def _attend(self, q, g0: int, g1: int, stream=None):
        st, s = self.step, self.s
        u0, u1 = g0 * self.group, g1 * self.group
        kernels.sparse_decode(q[u0:u1], self.pool_k[u0:u1], self.pool_v[u0:u1], idx=self.idx_pool[u0:u1],
                              cnt=st.cnt[u0:u1], causal_base=s.context - self.shift, rows_per_head=s.rows,
                              out=st.out[u0:u1], lse=st.lse[u0:u1], status=st.status, workspace=st.ws_dec,
                              stream=stream)

    def attend_on_demand(self, q):
        """Copy a layer's pages, attend it, next layer (one stream, serialised)."""
        self.plan()
        for g in range(self.groups):
            self._copy(g, g + 1)
            self._attend(q, g, g + 1)
        return self.step.out

    def attend_prefetch(self, q, layers_per_group: int = 1):
        """All layers' pages queued on the copy stream at once (the masks are
        known before layer 0); a group of ``layers_per_group`` layers attends
        when its pages have landed.  Per-layer groups overlap the most link
        time; when few pages move (a warm resident pool) larger groups save
        the per-group launch and cross-stream waits."""
        main = torch.cuda.current_stream(self.step.device)
        self.plan()
        self.copy_stream.wait_stream(main)
        lg = max(1, int(layers_per_group))
        bounds = [(g, min(g + lg, self.groups)) for g in range(0, self.groups, lg)]
        events = []
        with torch.cuda.stream(self.copy_stream):
            for g0, g1 in bounds:
                self._copy(g0, g1)
                e = torch.cuda.Event()
                e.record(self.copy_stream)
                events.append(e)
        for (g0, g1), e in zip(bounds, events):
            main.wait_event(e)
            self._attend(q, g0, g1)
        return self.step.out

    def bytes_moved(self) -> int:
        """Host-link bytes of the last plan (K + V of every copied page,
        committed pages plus the in-block tail)."""
        npg = int(self.npages.sum().item()) + self.U * (self.pages_ld - self.tail_rank0)
        return npg * self.P * self.d * self.hk.element_size() * 2

    def reset(self):
        """Empty the resident pool (the next step copies every page)."""
        if self.resident:
            self.slot_page.fill_(-1)
            self.slot_last.fill_(-1)
            self.step_no = 0
