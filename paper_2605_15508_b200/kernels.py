"""Batched tensor entry points over the C-ABI (torch tensors in, torch out).

These are the B200-native batched forms of the reference hot-path functions;
the reference-named, dict-of-numpy API in ``sparsity.py`` is built on them.
torch is used only for device memory and streams.  Every function launches
native kernels from libsts_b200.so; none of them computes on the CPU.
"""

from __future__ import annotations

import math

import torch

from . import _lib
from ._lib import call, ptr, stream_handle

STS_DTYPE = {torch.float32: _lib.STS_DTYPE_F32, torch.bfloat16: _lib.STS_DTYPE_BF16}
SCHEDULES = (0, 1, 2, 3, 4, 6, 8)  # bf16 decode work schedules (see sparse_decode)


def _require_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("tensor must live on a CUDA device (no CPU path exists)")


def _require_kv(*ts, host_kv=False):
    """K/V caches live in HBM, or (host_kv=True, the offload tier) in pinned,
    device-mapped host memory that the kernels read over the host link."""
    for t in ts:
        if t is None:
            continue
        if t.is_cuda:
            continue
        if host_kv and t.is_pinned():
            continue
        raise ValueError("K/V must be CUDA tensors (or pinned host tensors with host_kv=True)")


class Workspace:
    """Grow-only device scratch buffer (allocate once, reuse every step)."""

    def __init__(self, device=None):
        self.device = device
        self.buf = None

    def get(self, nbytes: int):
        if nbytes <= 0:
            return None, 0
        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = torch.empty(int(nbytes), dtype=torch.uint8, device=self.device or "cuda")
        return self.buf, self.buf.numel()


_DEFAULT_WS = {}


def _ws(key, device):
    w = _DEFAULT_WS.get((key, str(device)))
    if w is None:
        w = _DEFAULT_WS[(key, str(device))] = Workspace(device)
    return w


def resolve_budget(budget) -> tuple[float, int]:
    """SparsityConfig.budget -> (value, is_fraction) (src/sparsity.py:62-66)."""
    if isinstance(budget, bool):
        raise TypeError("budget must be int or float")
    if isinstance(budget, int):
        return float(budget), 0
    return float(budget), 1


def index_capacity(max_len: int, budget, page_size: int = 1, include_current=True,
                   include_sink=False, recent_window=0, tail_len=0) -> int:
    """Upper bound of one selection's index count (the idx_ld to allocate)."""
    value, frac = resolve_budget(budget)
    b = max(1, math.ceil(value * max_len)) if frac else int(value)
    sel = min(max_len, -(-b // page_size) * page_size + int(include_current) + int(include_sink)
              + int(recent_window))
    return max(1, sel + int(tail_len))


def select_topk(scores: torch.Tensor, *, budget, page_size: int = 1, include_current: bool = True,
                include_sink: bool = False, recent_window: int = 0, row_len=None, n_common=None,
                row_src=None, tail_len: int = 0, idx_ld=None, out=None, cnt=None, status=None,
                workspace: Workspace | None = None, stream=None):
    """Top-k / top-pages index masks of (reduced) score rows on the GPU.

    scores: fp32 [S, ld] device rows.  Logical rows are either the score rows
    themselves (row_src None) or fp32 sums of row_src[r, :] source rows.
    Returns (idx int32 [rows, idx_ld], cnt int32 [rows]); row r's mask is
    idx[r, :cnt[r]], ascending.  Semantics: include/sts_b200.h sts_select_topk.
    """
    _require_cuda(scores)
    if scores.dtype != torch.float32 or scores.dim() != 2 or scores.stride(1) != 1:
        raise ValueError("scores must be a row-major fp32 [S, ld] tensor")
    ld = scores.stride(0)
    if row_src is not None:
        row_src = row_src.to(device=scores.device, dtype=torch.int32).contiguous()
        rows, nsrc = row_src.shape
    else:
        rows, nsrc = scores.shape[0], 1
    if row_len is not None:
        row_len = row_len.to(device=scores.device, dtype=torch.int32).contiguous()
        max_len = ld
        n_common = 0
    else:
        n_common = scores.shape[1] if n_common is None else int(n_common)
        max_len = n_common
    value, frac = resolve_budget(budget)
    if idx_ld is None:
        idx_ld = index_capacity(max_len, budget, page_size, include_current, include_sink,
                                recent_window, tail_len)
    dev = scores.device
    if out is None:
        out = torch.empty((rows, idx_ld), dtype=torch.int32, device=dev)
    if cnt is None:
        cnt = torch.empty((rows,), dtype=torch.int32, device=dev)
    flags = (_lib.STS_SEL_CURRENT if include_current else 0) | (_lib.STS_SEL_SINK if include_sink else 0)
    lib = _lib.load()
    wbytes = lib.sts_select_workspace_bytes(rows, max_len, page_size)
    ws = workspace or _ws("select", dev)
    wbuf, wlen = ws.get(wbytes)
    call("sts_select_topk", ptr(scores), ld, ptr(row_src), nsrc, rows, ptr(row_len), n_common,
         value, frac, page_size, flags, recent_window, tail_len, ptr(out), out.stride(0), ptr(cnt),
         ptr(status), ptr(wbuf), wlen, stream_handle(stream))
    return out, cnt


def sparse_decode(q: torch.Tensor, k_cache: torch.Tensor, v_cache: torch.Tensor, *, idx=None,
                  cnt=None, n_dense: int = 0, member=None, causal_base: int = -1,
                  rows_per_head: int = 1, pos_offset: int = 0, scale=None, splits=None, schedule: int = 0,
                  out=None,
                  lse=None, status=None, out_dtype=None, host_kv: bool = False, workspace: Workspace | None = None,
                  stream=None):
    """Gathered-KV sparse flash-decode.

    q: [U, M, d] (bf16 or fp32); k_cache/v_cache: [U, N, d] views of the same
    dtype with unit inner stride (row stride >= d: an interleaved K|V cache
    [U, N, 2, d] passes kv[..., 0, :] and kv[..., 1, :]).  idx/cnt: int32 [U, ld] / [U] key lists
    (None => dense keys 0..n_dense-1).  Returns (out [U, M, d] q.dtype,
    lse fp32 [U, M]).  Semantics: include/sts_b200.h sts_sparse_decode.
    ``host_kv``: the caches may be pinned host tensors (KV offload tier): the
    same kernel then gathers only the selected rows over the host link.
    ``splits``: fp32 split-K factor.  ``schedule`` (bf16): 0 = auto (one
    thread-block cluster per unit for short key streams, else persistent
    stream-K), 1 = stream-K, 2/3/4/6/8 = clusters of that many CTAs per unit.
    """
    _require_cuda(q, idx, cnt, member)
    _require_kv(k_cache, v_cache, host_kv=host_kv)
    if q.dtype not in STS_DTYPE or k_cache.dtype != q.dtype or v_cache.dtype != q.dtype:
        raise ValueError("q, k_cache, v_cache must share dtype float32 or bfloat16")
    U, M, d = q.shape
    q = q.contiguous()
    if k_cache.stride(-1) != 1 or k_cache.stride(-2) < d or v_cache.stride() != k_cache.stride():
        raise ValueError("k_cache/v_cache must be [U, N, d] views with unit inner stride and equal strides")
    kv_stride = k_cache.stride(0)
    row_stride = k_cache.stride(1)
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    idx_ld = idx.stride(0) if idx is not None else 0
    if member is not None and (member.stride(0) != idx_ld or member.dtype != torch.int32 and member.dtype != torch.uint32):
        raise ValueError("member must be int32/uint32 with the same row stride as idx")
    if q.dtype == torch.bfloat16:
        # bf16: the argument is the work schedule (0 auto, 1 stream-K, C clusters of C CTAs per unit)
        if int(schedule) not in SCHEDULES:
            raise ValueError(f"schedule must be one of {SCHEDULES}")
        splits = int(schedule)
    elif splits is None:
        splits = 1
    dev = q.device
    out_dtype = q.dtype if out_dtype is None else out_dtype
    if out_dtype not in (q.dtype, torch.float32):
        raise ValueError("out_dtype must be q.dtype or float32")
    if out is None:
        out = torch.empty((U, M, d), dtype=out_dtype, device=dev)
    elif out.dtype != out_dtype:
        raise ValueError(f"out must be {out_dtype}")
    if lse is None:
        lse = torch.empty((U, M), dtype=torch.float32, device=dev)
    lib = _lib.load()
    wbytes = lib.sts_sparse_decode_workspace_bytes(U, M, d, splits)
    ws = workspace or _ws("decode", dev)
    wbuf, wlen = ws.get(wbytes)
    call("sts_sparse_decode", STS_DTYPE[q.dtype], STS_DTYPE[out_dtype], ptr(q), ptr(k_cache), ptr(v_cache), kv_stride, row_stride, U, M,
         d, ptr(idx), idx_ld, ptr(cnt), int(n_dense), ptr(member), int(causal_base), int(rows_per_head),
         int(pos_offset), scale, ptr(out), ptr(lse), int(splits), ptr(status), ptr(wbuf), wlen,
         stream_handle(stream))
    return out, lse


def kv_prefetch_l2(k_cache: torch.Tensor, v_cache: torch.Tensor, *, idx=None, cnt, parts: int = 1,
                   keys_per_part: int, stream=None):
    """Prefetch into L2 the K/V rows of the first ``keys_per_part`` keys of
    each of ``parts`` contiguous shares of every unit's key list
    (sts_kv_prefetch_l2). No output; nothing depends on it for correctness."""
    _require_cuda(k_cache, v_cache, idx, cnt)
    U, _, d = k_cache.shape
    if k_cache.stride(-1) != 1 or v_cache.stride() != k_cache.stride():
        raise ValueError("k_cache/v_cache must be [U, N, d] views with unit inner stride and equal strides")
    call("sts_kv_prefetch_l2", ptr(k_cache), ptr(v_cache), k_cache.stride(0), k_cache.stride(1), U, d,
         k_cache.element_size(), ptr(idx), idx.stride(0) if idx is not None else 0, ptr(cnt), int(parts),
         int(keys_per_part), stream_handle(stream))


def sparse_prefill(q: torch.Tensor, k_cache: torch.Tensor, v_cache: torch.Tensor, *, idx, cnt, scale=None,
                   out=None, lse=None, out_dtype=None, status=None, workspace: Workspace | None = None, stream=None):
    """Sparse prefill attention (STS-PD): every query row has its own key list.

    q: [G, n, M, d] (G K/V blocks, n query rows, M heads sharing block g and
    the row's mask; M = 1 for MHA); k_cache/v_cache: [G, N, d] views (unit
    inner stride); idx/cnt: int32 [G*n, ld] / [G*n] per-row key lists (causal
    by construction).  Returns (out [G, n, M, d], lse fp32 [G, n, M]).
    Semantics: include/sts_b200.h sts_sparse_prefill.
    """
    _require_cuda(q, k_cache, v_cache, idx, cnt)
    if q.dtype not in STS_DTYPE or k_cache.dtype != q.dtype or v_cache.dtype != q.dtype:
        raise ValueError("q, k_cache, v_cache must share dtype float32 or bfloat16")
    G, n, M, d = q.shape
    q = q.contiguous()
    if k_cache.stride(-1) != 1 or v_cache.stride() != k_cache.stride():
        raise ValueError("k_cache/v_cache must be [G, N, d] views with unit inner stride and equal strides")
    if idx.shape[0] != G * n or cnt.shape[0] != G * n:
        raise ValueError("idx/cnt need one row per (block, query row)")
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    out_dtype = q.dtype if out_dtype is None else out_dtype
    dev = q.device
    if out is None:
        out = torch.empty((G, n, M, d), dtype=out_dtype, device=dev)
    if lse is None:
        lse = torch.empty((G, n, M), dtype=torch.float32, device=dev)
    lib = _lib.load()
    wbytes = lib.sts_sparse_decode_workspace_bytes(G * n, M, d, 1)
    ws = workspace or _ws("decode", dev)
    wbuf, wlen = ws.get(wbytes)
    call("sts_sparse_prefill", STS_DTYPE[q.dtype], STS_DTYPE[out_dtype], ptr(q), ptr(k_cache), ptr(v_cache),
         k_cache.stride(0), k_cache.stride(1), G, n, M, d, ptr(idx), idx.stride(0), ptr(cnt), scale, ptr(out),
         ptr(lse), ptr(status), ptr(wbuf), wlen, stream_handle(stream))
    return out, lse


def draft_lse(q: torch.Tensor, k_cache: torch.Tensor, *, G: int, R: int, base: int, n_keys=None,
              pos_offset: int = 0, scale=None, out=None, workspace: Workspace | None = None,
              stream=None):
    """Natural-log LSE of each draft row (q [U, G*R, d] bf16, k_cache [U, N, d])."""
    _require_cuda(q, k_cache)
    U, GR, d = q.shape
    n_keys = k_cache.shape[1] if n_keys is None else int(n_keys)
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    if out is None:
        out = torch.empty((U, GR), dtype=torch.float32, device=q.device)
    lib = _lib.load()
    ws = workspace or _ws("draft", q.device)
    wbuf, wlen = ws.get(lib.sts_draft_workspace_bytes(U, GR, n_keys))
    call("sts_draft_lse", STS_DTYPE[q.dtype], ptr(q.contiguous()), ptr(k_cache), k_cache.stride(0), U,
         G, R, d, n_keys, pos_offset, base, scale, ptr(out), ptr(wbuf), wlen, stream_handle(stream))
    return out


def draft_probs(q: torch.Tensor, k_cache: torch.Tensor, lse: torch.Tensor, *, G: int, R: int,
                base: int, mode: str = "S", n_keys=None, pos_offset: int = 0, scale=None, out=None,
                stream=None):
    """Draft attention probabilities: mode "S" -> [U*G, ld] rows summed over the
    R speculative rows (committed positions only); mode "R" -> [U*G*R, ld]
    per-row probabilities (row i valid up to global position base+i)."""
    _require_cuda(q, k_cache, lse)
    U, GR, d = q.shape
    n_keys = k_cache.shape[1] if n_keys is None else int(n_keys)
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    m = 0 if mode == "S" else 1
    if out is None:
        rows = U * G if m == 0 else U * GR
        out = torch.zeros((rows, n_keys), dtype=torch.float32, device=q.device)
    call("sts_draft_probs", STS_DTYPE[q.dtype], ptr(q.contiguous()), ptr(k_cache), k_cache.stride(0),
         U, G, R, d, n_keys, pos_offset, base, scale, ptr(lse), m, ptr(out), out.stride(0),
         stream_handle(stream))
    return out


def draft_scores(q: torch.Tensor, k_cache: torch.Tensor, *, G: int, R: int, base: int, n_keys=None,
                 pos_offset: int = 0, scale=None, out=None, stream=None):
    """Raw draft scores (the reference's ForwardRecord.scores, src/toymodel.py:
    225-240, :351-352): [U*G*R, ld] fp32 rows of scale * q.k, row i valid up to
    global position base+i (the rest stays as allocated: zeros by default)."""
    _require_cuda(q, k_cache)
    U, GR, d = q.shape
    n_keys = k_cache.shape[1] if n_keys is None else int(n_keys)
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    if out is None:
        out = torch.zeros((U * GR, n_keys), dtype=torch.float32, device=q.device)
    call("sts_draft_scores", STS_DTYPE[q.dtype], ptr(q.contiguous()), ptr(k_cache), k_cache.stride(0), U, G, R, d,
         n_keys, pos_offset, base, scale, ptr(out), out.stride(0), stream_handle(stream))
    return out


def lse_merge(o_parts: torch.Tensor | None, lse_parts: torch.Tensor, *, out_dtype=torch.float32,
              out=None, lse_out=None, stream=None):
    """Merge P partial attention results: o_parts [P, rows, d] fp32 (or None),
    lse_parts [P, rows] -> (out [rows, d], lse [rows])."""
    _require_cuda(lse_parts)
    P, rows = lse_parts.shape
    d = o_parts.shape[-1] if o_parts is not None else 1
    if out is None and o_parts is not None:
        out = torch.empty((rows, d), dtype=out_dtype, device=lse_parts.device)
    if lse_out is None:
        lse_out = torch.empty((rows,), dtype=torch.float32, device=lse_parts.device)
    call("sts_lse_merge", ptr(o_parts), ptr(lse_parts.contiguous()), P, rows, d, STS_DTYPE[out_dtype],
         ptr(out), ptr(lse_out), stream_handle(stream))
    return out, lse_out


def row_union(idx, cnt, src, *, M: int, n_max: int, out_ld=None, bitmap=None, status=None,
              stream=None):
    """Mode-R union: per unit, merge its M source lists (src [U, M] rows of
    idx/cnt) into one ascending list + per-key row-membership bits."""
    _require_cuda(idx, cnt, src)
    src = src.to(device=idx.device, dtype=torch.int32).contiguous()
    U = src.shape[0]
    out_ld = n_max if out_ld is None else out_ld
    dev = idx.device
    if bitmap is None:
        bitmap = torch.empty((U, n_max), dtype=torch.int32, device=dev)
    idx_out = torch.empty((U, out_ld), dtype=torch.int32, device=dev)
    member = torch.empty((U, out_ld), dtype=torch.int32, device=dev)
    cnt_out = torch.empty((U,), dtype=torch.int32, device=dev)
    call("sts_row_union", ptr(idx), idx.stride(0), ptr(cnt), ptr(src), U, M, n_max, ptr(bitmap),
         ptr(idx_out), ptr(member), out_ld, ptr(cnt_out), ptr(status), stream_handle(stream))
    return idx_out, member, cnt_out


PREFILL_TILE = 128   # query rows per tile of the block-sparse prefill
PREFILL_BLOCK = 64   # keys per selectable block


def prefill_tile_select(tile_scores: torch.Tensor, *, budget, n: int, out=None, cnt=None, status=None,
                        workspace: Workspace | None = None, stream=None):
    """Block selection of the block-sparse prefill: for every (kv-head, query
    tile T) score row (fp32 [Hkv * tiles, ld], keys = positions), the top
    ``ceil(b / 64)`` 64-key blocks among the committed positions [0, 128 T)
    (budget b of that context, src/sparsity.py:62-66, numkit tie rule), as
    whole blocks of ascending tokens.  Tile 0 has no committed blocks."""
    tiles = -(-n // PREFILL_TILE)
    rows = tile_scores.shape[0]
    if rows % tiles:
        raise ValueError("tile_scores must hold heads_kv * tiles rows")
    T = torch.arange(tiles, dtype=torch.int32, device=tile_scores.device).repeat(rows // tiles)
    row_len = torch.clamp(T * PREFILL_TILE, min=1)
    idx, cnt = select_topk(tile_scores, budget=budget, page_size=PREFILL_BLOCK, include_current=False,
                           row_len=row_len, out=out, cnt=cnt, status=status, workspace=workspace, stream=stream)
    cnt.masked_fill_(T == 0, 0)
    return idx, cnt


def prefill_blocksparse(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, *, idx=None, cnt=None, scale=None,
                        out=None, status=None, stream=None):
    """Block-sparse causal prefill on tcgen05 (include/sts_b200.h
    sts_prefill_blocksparse): q [Hq, n, d], k/v [Hkv, n, d] bf16 (unit inner
    stride, rows 16-byte aligned); idx/cnt from ``prefill_tile_select`` (None:
    dense causal).  Returns out [Hq, n, d] bf16."""
    _require_cuda(q, k, v, idx, cnt)
    if q.dtype != torch.bfloat16 or k.dtype != torch.bfloat16 or v.dtype != torch.bfloat16:
        raise ValueError("block-sparse prefill runs on bf16 q / k / v")
    Hq, n, d = q.shape
    Hkv = k.shape[0]
    if k.shape != (Hkv, n, d) or v.stride() != k.stride() or q.stride(1) != k.stride(1):
        raise ValueError("q [Hq, n, d] and k/v [Hkv, n, d] must share the row stride")
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    if out is None:
        out = torch.empty((Hq, n, d), dtype=torch.bfloat16, device=q.device)
    call("sts_prefill_blocksparse", ptr(q), ptr(k), ptr(v), Hq, Hkv, n, d, q.stride(0), k.stride(0), k.stride(1),
         scale, ptr(idx), idx.stride(0) if idx is not None else 0, ptr(cnt), ptr(out), ptr(status),
         stream_handle(stream))
    return out
