"""CPU oracle for the STS sparse-attention hot path — TEST INFRASTRUCTURE ONLY.

This module is the parity checker. Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.
The product package (``paper_2605_15508_b200``) never imports it and never
falls back to it.

It restates, in numpy, the reference package ``specsparse`` (arxiv
2605.15508 desk-scale lab, ``/root/reference/pkg/src/specsparse``) for the
hot path, function by function, citing the reference file:line each follows.
Parity is PINNED: ``tests/golden/make_golden.py`` imports the real reference
in the build container and records its outputs on seeded inputs into
``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` checks every function
here against those vectors and against the reference's own known-answer tests
(``pkg/tests/test_numkit.py:86-113``, ``pkg/tests/test_sparsity.py:31-235``).

Sections:
  1. reference restatements (MHA, per row, fp64 compute)      — reference-exact
  2. mode-S restatement (rows reduced over speculative queries and the GQA
     group)                              — new, defined here
  3. sequence-sharded selection + LSE merge                   — new, defined here
  4. key ordering used by the GPU radix select (documentation + checker)
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

# ---------------------------------------------------------------------------
# errors (mirror src/errors.py:11-44; the oracle raises the same *names*)
# ---------------------------------------------------------------------------


class OracleContractViolation(Exception):
    """Mirror of specsparse.errors.ContractViolation (src/errors.py:19)."""


class OracleConfigError(Exception):
    """Mirror of specsparse.errors.ConfigError (src/errors.py:27)."""


# ---------------------------------------------------------------------------
# 1. reference restatements
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class OracleSparsityConfig:
    """src/sparsity.py:33-69 (SparsityConfig)."""

    budget: float
    page_size: int = 1
    include_current: bool = True
    include_sink: bool = False
    recent_window: int = 0

    def tokens_for_context(self, n: int) -> int:
        """src/sparsity.py:62-66: int budget is absolute; float is max(1, ceil(f*n))."""
        if isinstance(self.budget, (int, np.integer)) and not isinstance(self.budget, bool):
            return int(self.budget)
        return max(1, math.ceil(self.budget * n))


def topk_indices(scores, k: int) -> np.ndarray:
    """src/numkit.py:74-86: k largest, ties -> lowest index, ascending output.

    fp32 inputs are promoted to fp64 exactly; ``np.argsort(kind="stable")`` on
    the negated array keeps the lowest index first among equal scores; NaN
    sorts after every number (so it ranks last), -0.0 == +0.0.
    """
    if k < 1:
        raise OracleContractViolation(f"k must be >= 1, got {k}")
    arr = np.asarray(scores, dtype=np.float64).ravel()
    if arr.size == 0:
        raise OracleContractViolation("cannot take top-k of an empty score list")
    order = np.argsort(-arr, kind="stable")[: min(k, arr.size)]
    return np.sort(order).astype(np.int64)


def page_aggregate(scores, page_size: int) -> np.ndarray:
    """src/sparsity.py:72-83: fp64 page sums, ragged last page.

    Summation order is numpy's ``add.reduceat``: ``x0 + pairwise(x[1:])``
    (see ``numpy_pairwise_sum`` below, which the tests pin against reduceat).
    """
    if page_size < 1:
        raise OracleContractViolation("page_size must be >= 1")
    arr = np.asarray(scores, dtype=np.float64).ravel()
    if page_size == 1:
        return arr.copy()
    edges = np.arange(0, arr.size, page_size)
    return np.add.reduceat(arr, edges)


def numpy_pairwise_sum(a) -> float:
    """Explicit restatement of numpy's float64 pairwise summation.

    numpy/_core/src/umath/loops_utils.h.src (``pairwise_sum``): n < 8 is a
    sequential sum from 0.0; 8 <= n <= 128 uses 8 strided accumulators
    combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) then a sequential tail;
    n > 128 splits at n2 = n/2 rounded down to a multiple of 8 and recurses.
    ``np.add.reduceat`` on a segment computes ``x[a] + pairwise(x[a+1:b])``.
    This is the order the CUDA page-sum device function reproduces.
    """
    a = np.asarray(a, dtype=np.float64)
    n = a.size
    if n < 8:
        res = np.float64(0.0)
        for v in a:
            res = res + v
        return res
    if n <= 128:
        r = [a[j] for j in range(8)]
        i = 8
        while i < n - (n % 8):
            for j in range(8):
                r[j] = r[j] + a[i + j]
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            res = res + a[i]
            i += 1
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return numpy_pairwise_sum(a[:n2]) + numpy_pairwise_sum(a[n2:])


def select_row(row, cfg: OracleSparsityConfig) -> np.ndarray:
    """src/sparsity.py:86-112 (_select_row): dense / top-k / top-pages + extras."""
    row = np.asarray(row)
    n = row.shape[0]
    budget = cfg.tokens_for_context(n)
    if budget >= n:
        selected = np.arange(n, dtype=np.int64)
    elif cfg.page_size == 1:
        selected = topk_indices(row, budget)
    else:
        pages = page_aggregate(row, cfg.page_size)
        top_pages = topk_indices(pages, math.ceil(budget / cfg.page_size))
        chunks = [
            np.arange(p * cfg.page_size, min((p + 1) * cfg.page_size, n), dtype=np.int64)
            for p in top_pages
        ]
        selected = np.concatenate(chunks)
    extras = []
    if cfg.include_current:
        extras.append(n - 1)
    if cfg.include_sink:
        extras.append(0)
    if cfg.recent_window > 0:
        extras.extend(range(max(0, n - cfg.recent_window), n))
    if extras:
        selected = np.union1d(selected, np.asarray(extras, dtype=np.int64))
    return np.sort(np.unique(selected))


def draft_masks_decode(rows: dict, cfg: OracleSparsityConfig) -> dict:
    """src/sparsity.py:115-119."""
    return {head: select_row(np.asarray(row), cfg) for head, row in rows.items()}


def draft_masks_prefill(matrices: dict, cfg: OracleSparsityConfig) -> dict:
    """src/sparsity.py:122-130: per causal row t over mat[t, :t+1]."""
    out = {}
    for head, mat in matrices.items():
        mat = np.asarray(mat)
        out[head] = [select_row(mat[t, : t + 1], cfg) for t in range(mat.shape[0])]
    return out


def remap_masks(draft_masks: dict, entries: dict) -> dict:
    """src/sparsity.py:133-149: target <- copy(mask[entries[target][0]])."""
    out = {}
    for target, (draft, _score) in entries.items():
        if draft not in draft_masks:
            raise OracleContractViolation(f"no draft mask for head {draft} (target {target})")
        value = draft_masks[draft]
        if isinstance(value, list):
            out[target] = [np.array(v, dtype=np.int64, copy=True) for v in value]
        else:
            out[target] = np.array(value, dtype=np.int64, copy=True)
    return out


def clamp_current(indices, pos: int) -> np.ndarray:
    """src/specdec.py:212-216 (_clamp_current)."""
    arr = np.asarray(indices, dtype=np.int64)
    arr = arr[arr <= pos]
    return np.union1d(arr, np.asarray([pos], dtype=np.int64))


def verification_masks(draft_rows: list, base: int, cfg: OracleSparsityConfig, entries: dict) -> dict:
    """src/specdec.py:219-233 (_verification_masks): per-row target masks."""
    per_row = []
    for i, rows in enumerate(draft_rows):
        masks = remap_masks(draft_masks_decode(rows, cfg), entries)
        per_row.append({h: clamp_current(m, base + i) for h, m in masks.items()})
    return {head: [per_row[i][head] for i in range(len(draft_rows))] for head in per_row[0]}


def nearest_mapping_k(ks, budget: int) -> int:
    """src/headmap.py:181-182 (MappingSet.nearest): min |k - budget|, ties -> smaller k."""
    return min(sorted(ks), key=lambda k: (abs(k - budget), k))


def sparse_attention(q, keys, values, mask) -> np.ndarray:
    """src/sparsity.py:152-173: fp64 gather-softmax-PV, fp32 result."""
    idx = np.asarray(mask, dtype=np.int64).ravel()
    if idx.size == 0:
        raise OracleContractViolation("sparse attention needs a non-empty mask")
    if idx.min() < 0 or idx.max() >= keys.shape[0]:
        raise OracleContractViolation("mask index outside the cached context")
    q64 = np.asarray(q, dtype=np.float64)
    k_sel = np.asarray(keys, dtype=np.float64)[idx]
    v_sel = np.asarray(values, dtype=np.float64)[idx]
    scores = (k_sel @ q64) / math.sqrt(q64.shape[0])
    scores -= scores.max()
    weights = np.exp(scores)
    weights /= weights.sum()
    return (weights @ v_sel).astype(np.float32)


def sparse_attention_lse(q, keys, values, mask):
    """sparse_attention plus the natural-log LSE of the scaled scores (fp64).

    The LSE is what the GPU kernels export for split/shard merging; the
    output half is identical to ``sparse_attention``.
    """
    idx = np.asarray(mask, dtype=np.int64).ravel()
    q64 = np.asarray(q, dtype=np.float64)
    k_sel = np.asarray(keys, dtype=np.float64)[idx]
    v_sel = np.asarray(values, dtype=np.float64)[idx]
    scores = (k_sel @ q64) / math.sqrt(q64.shape[0])
    mx = scores.max()
    w = np.exp(scores - mx)
    s = w.sum()
    return (w / s) @ v_sel, mx + math.log(s)


def draft_attention_rows(q, keys, base: int, rows: int):
    """Draft score capture, src/toymodel.py:315-352 as reached from
    specdec.propose (src/specdec.py:150-167): row i (query at position base+i)
    is softmax(q_i . K[0..base+i] / sqrt(d)) in fp64, recorded as fp32.

    q: (rows, d); keys: (>= base+rows, d). Returns list of fp32 rows, row i of
    length base+i+1.
    """
    d = q.shape[-1]
    out = []
    k64 = np.asarray(keys, dtype=np.float64)
    for i in range(rows):
        n = base + i + 1
        s = (k64[:n] @ np.asarray(q[i], dtype=np.float64)) * (1.0 / math.sqrt(d))
        s -= s.max()
        w = np.exp(s)
        w /= w.sum()
        out.append(w.astype(np.float32))
    return out


# ---------------------------------------------------------------------------
# 2. mode S (shared / reduced) restatement — SURVEY Appendix A.5, DESIGN.md §3
# ---------------------------------------------------------------------------


def reduce_rows_fp32(rows_list) -> np.ndarray:
    """Sequential fp32 sum in list order: ((r0 + r1) + r2) + ...

    Used for (a) the GPU draft kernel's row reduction D = sum_i p_i (checked by
    tolerance, since the p_i themselves come from expf) and (b) the select
    kernel's head-group reduction r = sum_h D[map(h)] (checked bit-exactly).
    """
    acc = np.zeros_like(np.asarray(rows_list[0], dtype=np.float32))
    for r in rows_list:
        acc = (acc + np.asarray(r, dtype=np.float32)).astype(np.float32)
    return acc


def select_committed(row, n: int, budget: int, cfg: OracleSparsityConfig) -> np.ndarray:
    """Mode-S selection over committed positions [0, n) with an explicit budget.

    Same recipe as select_row (src/sparsity.py:86-112) but the budget is
    supplied (tokens_for_context(base+1), the per-round budget specdec uses
    for its mapping choice, src/specdec.py:331) and ``include_current`` is not
    applied: in mode S every verify row attends its own in-block position via
    the causal tail, so the committed-range extras are sink + recent window.
    """
    row = np.asarray(row)[:n]
    if budget >= n:
        selected = np.arange(n, dtype=np.int64)
    elif cfg.page_size == 1:
        selected = topk_indices(row, budget)
    else:
        pages = page_aggregate(row, cfg.page_size)
        top_pages = topk_indices(pages, math.ceil(budget / cfg.page_size))
        selected = np.concatenate([
            np.arange(p * cfg.page_size, min((p + 1) * cfg.page_size, n), dtype=np.int64)
            for p in top_pages
        ])
    extras = []
    if cfg.include_sink:
        extras.append(0)
    if cfg.recent_window > 0:
        extras.extend(range(max(0, n - cfg.recent_window), n))
    if extras:
        selected = np.union1d(selected, np.asarray(extras, dtype=np.int64))
    return np.sort(np.unique(selected))


def mode_s_index_list(reduced_row, base: int, tail: int, cfg: OracleSparsityConfig) -> np.ndarray:
    """Full mode-S key list for one (layer, kv-group): committed selection
    followed by the in-block positions base .. base+tail-1 (ascending)."""
    budget = cfg.tokens_for_context(base + 1)
    sel = select_committed(reduced_row, base, budget, cfg) if base > 0 else np.zeros(0, np.int64)
    return np.concatenate([sel, np.arange(base, base + tail, dtype=np.int64)])


def block_attention(q_rows, keys, values, idx, causal_base=None, rows_per_head=1, member=None):
    """Attention of M stacked query rows over one shared key list (fp64).

    Row r attends key idx[j] iff (causal_base is None or idx[j] - causal_base
    <= r % rows_per_head) and (member is None or bit r of member[j]).
    Returns (out fp64 (M, d), lse fp64 (M,)).
    """
    idx = np.asarray(idx, dtype=np.int64)
    return block_attention_rows(q_rows, np.asarray(keys)[idx], np.asarray(values)[idx], idx, causal_base,
                                rows_per_head, member)


def block_attention_rows(q_rows, k_sel, v_sel, positions, causal_base=None, rows_per_head=1, member=None):
    """block_attention over already-gathered key/value rows: k_sel[j], v_sel[j]
    sit at cache position positions[j] (the causal test uses the positions)."""
    q = np.asarray(q_rows, dtype=np.float64)
    M, d = q.shape
    idx = np.asarray(positions, dtype=np.int64)
    k = np.asarray(k_sel, dtype=np.float64)
    v = np.asarray(v_sel, dtype=np.float64)
    s = (q @ k.T) / math.sqrt(d)
    allowed = np.ones_like(s, dtype=bool)
    r = np.arange(M)
    if causal_base is not None:
        allowed &= (idx[None, :] - causal_base) <= (r % rows_per_head)[:, None]
    if member is not None:
        mem = np.asarray(member, dtype=np.uint64)
        allowed &= ((mem[None, :] >> r[:, None].astype(np.uint64)) & np.uint64(1)).astype(bool)
    s = np.where(allowed, s, -np.inf)
    mx = s.max(axis=1, keepdims=True)
    w = np.exp(s - mx)
    w[~allowed] = 0.0
    tot = w.sum(axis=1, keepdims=True)
    return (w / tot) @ v, (mx[:, 0] + np.log(tot[:, 0]))


# ---------------------------------------------------------------------------
# 3. sequence-sharded selection and LSE merge
# ---------------------------------------------------------------------------


def shard_bounds(n: int, nranks: int, align: int = 1):
    """Contiguous, ``align``-aligned token ranges [lo, hi) per rank."""
    per = -(-n // nranks)
    per = -(-per // align) * align
    return [(min(r * per, n), min((r + 1) * per, n)) for r in range(nranks)]


def lse_merge(outs, lses):
    """LSE = log sum exp(LSE_r); O = sum exp(LSE_r - LSE) O_r (fp64)."""
    lses = np.asarray(lses, dtype=np.float64)
    m = np.max(lses, axis=0)
    w = np.exp(lses - m)
    tot = w.sum(axis=0)
    out = sum(w[r][..., None] * np.asarray(outs[r], dtype=np.float64) for r in range(len(outs)))
    return out / tot[..., None], m + np.log(tot)


# ---------------------------------------------------------------------------
# 4. key ordering of the GPU radix select
# ---------------------------------------------------------------------------


def fp32_order_keys(x) -> np.ndarray:
    """uint32 keys whose unsigned order equals the reference's rank order.

    -0.0 is canonicalised to +0.0; NaN maps to 0 (ranks below -inf); ties
    between equal keys are then broken by the lower index, exactly as the
    stable argsort in src/numkit.py:84 does on fp64-promoted fp32 values.
    """
    x = np.asarray(x, dtype=np.float32) + np.float32(0.0)
    b = x.view(np.uint32)
    keys = np.where(b >> 31 == 1, ~b, b | np.uint32(0x80000000)).astype(np.uint32)
    keys[np.isnan(x)] = 0
    return keys


# ---------------------------------------------------------------------------
# 5. sequence-sharded radix-select protocol (restates csrc/sts_select_dist.cu)
# ---------------------------------------------------------------------------

DIST_BITS = 11  # digit width (the last digit takes the remaining bits)


def dist_digits(kbits: int = 32):
    """(shift, width) of each radix round, from the top (csrc/sts_select_dist.cu dd_*)."""
    out, top = [], kbits
    while top > 0:
        w = min(DIST_BITS, top)
        out.append((top - w, w))
        top -= w
    return out


def dist_select_protocol(values_local, lo: int, n_global: int, k: int, rank: int, nranks: int, torch_mod=None):
    """One rank of the sharded top-k protocol, in numpy, yielding the same
    collective requests as paper_2605_15508_b200.sharded.DistSelector
    (("all_reduce_sum", int32 tensor [rows][2048]), ("all_gather", ties [rows],
    ties_all [P][rows])).  Returns the selected GLOBAL indices per row
    (ascending).  ``values_local``: fp32 [rows, n_local] at global positions
    lo.. ; positions >= n_global are ignored.  Token mode, fp32 keys, 11-bit
    digits from the top (11 + 11 + 10); the threshold/tie rule of topk_indices
    (src/numkit.py:74-86)."""
    import torch

    vals = np.asarray(values_local, dtype=np.float32)
    rows = vals.shape[0]
    nc = max(0, min(n_global - lo, vals.shape[1]))
    keys = fp32_order_keys(vals[:, :nc]).astype(np.uint64) if nc else np.zeros((rows, 0), np.uint64)
    prefix = np.zeros(rows, np.uint64)
    pmask = np.zeros(rows, np.uint64)
    krem = np.full(rows, k, np.int64)
    dense = k >= n_global
    done = np.full(rows, dense, bool)
    ties_local = np.zeros(rows, np.int64)
    for shift, width in dist_digits(32):
        nb = 1 << width
        hist = np.zeros((rows, 1 << DIST_BITS), np.int64)
        for r in range(rows):
            if done[r]:
                continue
            m = (keys[r] & pmask[r]) == prefix[r]
            d = ((keys[r][m] >> np.uint64(shift)) & np.uint64(nb - 1)).astype(np.int64)
            hist[r, :nb] = np.bincount(d, minlength=nb)
        h_local = hist.copy()
        t = torch.from_numpy(hist.astype(np.int32))
        yield ("all_reduce_sum", t)
        hg = t.numpy().astype(np.int64)
        for r in range(rows):
            if done[r]:
                continue
            acc = 0
            for digit in range(nb - 1, -1, -1):
                c = int(hg[r, digit])
                if acc < krem[r] <= acc + c:
                    break
                acc += c
            prefix[r] |= np.uint64(digit) << np.uint64(shift)
            pmask[r] |= np.uint64(nb - 1) << np.uint64(shift)
            krem[r] -= acc
            if shift == 0 or krem[r] == c:
                done[r] = True
                ties_local[r] = h_local[r, digit]
    tl = torch.from_numpy(ties_local.astype(np.int32))
    ta = torch.zeros((nranks, rows), dtype=torch.int32)
    yield ("all_gather", tl, ta)
    ties_all = ta.numpy().astype(np.int64)
    out = []
    for r in range(rows):
        if dense:
            out.append(lo + np.arange(nc, dtype=np.int64))
            continue
        mk = keys[r] & pmask[r]
        above = mk > prefix[r]
        tie = mk == prefix[r]
        need = max(int(krem[r]) - int(ties_all[:rank, r].sum()), 0)
        take = np.zeros(nc, bool)
        take[np.nonzero(tie)[0][:need]] = True
        out.append(lo + np.nonzero(above | take)[0].astype(np.int64))
    return out


# ---------------------------------------------------------------------------
# 6. Algorithm 1 (src/headmap.py:59-125): best-overlap draft head per target
# ---------------------------------------------------------------------------


def rowwise_topk_sets(matrix, k: int):
    """src/headmap.py:59-62: top-k of each row's causal prefix."""
    n = matrix.shape[0]
    return [topk_indices(matrix[t, : t + 1], k) for t in range(n)]


def find_head_mapping(samples, draft_heads, target_heads, k: int) -> dict:
    """src/headmap.py:83-125 with python-set intersections (the reference
    uses integer bitmasks; the counts are the same).  samples: list of
    (draft dict, target dict).  Returns {target head: (draft head, score)}."""
    totals = {th: np.zeros(len(draft_heads), dtype=np.int64) for th in target_heads}
    for draft, target in samples:
        dsets = {dh: [set(s.tolist()) for s in rowwise_topk_sets(draft[dh], k)] for dh in draft_heads}
        for th in target_heads:
            tsets = [set(s.tolist()) for s in rowwise_topk_sets(target[th], k)]
            for j, dh in enumerate(draft_heads):
                totals[th][j] += sum(len(a & b) for a, b in zip(tsets, dsets[dh]))
    out = {}
    for th in target_heads:
        best = int(np.argmax(totals[th]))
        out[th] = (draft_heads[best], int(totals[th][best]))
    return out


# ---------------------------------------------------------------------------
# 5. toy-model weights (test fixtures for the model-level drop-in)
# ---------------------------------------------------------------------------


def lru_prefetch_steps(traces, capacity: int):
    """The "prefetch" strategy's residency for one layer
    (src/offloadsim.py:173-209 with _lru_insert / _lru_touch :135-150): per
    step, the pages not resident (in trace order) are inserted FIFO, evicting
    the first non-pinned page in LRU-dict order while the tier is full; then
    every page of the step is touched in trace order.  Returns per step the
    list of missing pages (what the device tier copies)."""
    resident: dict = {}
    out = []
    for pages in traces:
        pinned = set(pages)
        if len(pinned) > capacity:
            raise ValueError("step needs more pages than the tier holds")
        missing = [p for p in pages if p not in resident]
        for key in missing:
            while len(resident) >= capacity:
                victim = next(k for k in resident if k not in pinned)
                resident.pop(victim)
            resident[key] = True
        for key in pages:
            resident.pop(key)
            resident[key] = True
        out.append(missing)
    return out


@dataclass(frozen=True)
class OracleModelConfig:
    """Fields of src/toymodel.py:38-57 ``ModelConfig``."""

    layers: int
    heads: int
    head_dim: int
    vocab: int
    max_seq: int
    page_size: int = 4
    mlp_ratio: int = 4
    seed: int = 0

    @property
    def hidden(self) -> int:
        return self.heads * self.head_dim

    def to_dict(self) -> dict:
        return {k: getattr(self, k) for k in ("layers", "heads", "head_dim", "vocab", "max_seq", "page_size",
                                               "mlp_ratio", "seed")}


@dataclass
class OracleModelWeights:
    """Field names of src/toymodel.py:89-104 ``ModelWeights``."""

    config: OracleModelConfig
    token_emb: np.ndarray
    pos_emb: np.ndarray
    attn_norm: np.ndarray
    wq: np.ndarray
    wk: np.ndarray
    wv: np.ndarray
    wo: np.ndarray
    mlp_norm: np.ndarray
    w_up: np.ndarray
    w_down: np.ndarray
    final_norm: np.ndarray
    lm_head: np.ndarray


def init_model(config: OracleModelConfig) -> OracleModelWeights:
    """src/toymodel.py:126-160: every parameter drawn, in field order, from one
    PCG64 stream seeded with ``config.seed`` (numkit.prng_stream,
    src/numkit.py:89-95); projections scaled by 1/sqrt(hidden), norms 1."""
    rng = np.random.Generator(np.random.PCG64(config.seed))
    h = config.hidden
    mh = config.mlp_ratio * h
    scale = 1.0 / math.sqrt(h)

    def draw(*shape, s=1.0):
        return (rng.standard_normal(shape) * s).astype(np.float32)

    return OracleModelWeights(
        config=config,
        token_emb=draw(config.vocab, h),
        pos_emb=draw(config.max_seq, h),
        attn_norm=np.ones((config.layers, h), dtype=np.float32),
        wq=draw(config.layers, h, h, s=scale),
        wk=draw(config.layers, h, h, s=scale),
        wv=draw(config.layers, h, h, s=scale),
        wo=draw(config.layers, h, h, s=scale),
        mlp_norm=np.ones((config.layers, h), dtype=np.float32),
        w_up=draw(config.layers, h, mh, s=scale),
        w_down=draw(config.layers, mh, h, s=scale),
        final_norm=np.ones(h, dtype=np.float32),
        lm_head=draw(h, config.vocab, s=scale),
    )
