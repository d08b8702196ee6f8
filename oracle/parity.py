"""Sampled-unit parity of a device verify step against the CPU oracle —
TEST INFRASTRUCTURE ONLY (imported by ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``; the product package never imports it).

A mode-S verify step (``STSVerifyStep`` or one ``ShardedVerifyStep`` rank)
leaves on the device: the draft probability rows it captured, the head-group
table ``row_src``, the key lists ``idx``/``cnt`` and the attention output.
For a sample of units this module pulls only what the oracle needs to the
host — the unit's source rows, its key list, the gathered K/V rows of the
oracle's own key list and the unit's queries — and checks

  * masks bit-exactly: ``idx[u, :cnt[u]]`` == ``sts_oracle.mode_s_index_list``
    of ``reduce_rows_fp32`` of the unit's draft rows (the select contract of
    SURVEY §7.3 hard part 1: selection is exact given identical fp32 rows;
    reference rule ``src/numkit.py:74-86``, ``src/sparsity.py:86-112``);
  * attention within the bf16 tolerance (2e-2, north star) against
    ``sts_oracle.block_attention_rows`` (fp64, the math of
    ``src/sparsity.py:152-173`` over the stacked rows).

Only sampled rows and gathered keys cross the host link, so this runs at the
measured configurations (c2 32K, c3 128K x batch 8, c4 1M) in seconds.
"""

from __future__ import annotations

import numpy as np

from . import sts_oracle as O

BF16_TOL = 2e-2


def sample_units(batch: int, layers: int, kv_heads: int, n: int, seed: int = 0) -> list[int]:
    """``n`` distinct unit ids (b, l, g) -> (b*layers + l)*kv_heads + g with
    every layer represented before any repeats (n >= layers covers them all)."""
    rng = np.random.default_rng(seed)
    U = batch * layers * kv_heads
    n = min(n, U)
    out, seen = [], set()
    order = list(rng.permutation(layers))
    while len(out) < n:
        for l in order:
            if len(out) >= n:
                break
            for _ in range(64):
                u = (int(rng.integers(batch)) * layers + int(l)) * kv_heads + int(rng.integers(kv_heads))
                if u not in seen:
                    break
            if u in seen:
                continue
            seen.add(u)
            out.append(u)
        if len(seen) >= U:
            break
    return sorted(out)


def oracle_config(cfg) -> O.OracleSparsityConfig:
    return O.OracleSparsityConfig(cfg.budget, cfg.page_size, False, cfg.include_sink, cfg.recent_window)


def expected_index_list(draft_rows, row_src, u: int, context: int, tail: int, cfg) -> np.ndarray:
    """The oracle's mode-S key list of unit u from the device draft rows."""
    import torch

    src = row_src[u].long()
    rows = draft_rows.index_select(0, src)[:, :context].cpu().numpy()
    red = O.reduce_rows_fp32(list(rows))
    return O.mode_s_index_list(red, context, tail, oracle_config(cfg))


def check_units(step, q, k, v, out, units, cfg=None, pos_offset: int = 0, tol: float = BF16_TOL) -> dict:
    """Parity of ``units`` of a finished mode-S step (device tensors in ``step``:
    draft_rows, row_src, idx, cnt; q [U, M, d], k/v [U, N, d] unit views,
    out [U, M, d]).  Returns {"units", "masks_bit_exact", "mask_mismatch_units",
    "max_abs_err", "tol", "attention_ok"}."""
    import torch

    s = step.shape
    cfg = cfg if cfg is not None else step.cfg
    R, base = s.rows, s.context
    idx_h = step.idx.index_select(0, torch.tensor(units, device=step.idx.device)).cpu().numpy()
    cnt_h = step.cnt.index_select(0, torch.tensor(units, device=step.cnt.device)).cpu().numpy()
    bad, max_err = [], 0.0
    for j, u in enumerate(units):
        want = expected_index_list(step.draft_rows, step.row_src, u, base, R, cfg)
        got = idx_h[j, : cnt_h[j]].astype(np.int64) + pos_offset
        if not np.array_equal(got, want):
            bad.append(int(u))
        pos = torch.from_numpy(want - pos_offset).to(k.device)
        ks = k[u].index_select(0, pos).float().cpu().numpy()
        vs = v[u].index_select(0, pos).float().cpu().numpy()
        ref, _ = O.block_attention_rows(q[u].float().cpu().numpy(), ks, vs, want, causal_base=base,
                                        rows_per_head=R)
        err = float(np.abs(out[u].float().cpu().numpy() - ref).max())
        max_err = max(max_err, err)
    return {"units": len(units), "masks_bit_exact": not bad, "mask_mismatch_units": bad[:8],
            "max_abs_err": round(max_err, 6), "tol": tol, "attention_ok": max_err <= tol}


def mask_agreement(step, draft_q, draft_k, units, cfg=None) -> dict:
    """Agreement of the device masks with masks built from fp64 reference
    draft rows (overlap as in evalkit.mask_recall,
    src/evalkit.py:40-96).  For each sampled unit the reference path is
    restated from the device's bf16 inputs: every mapped draft head's γ+1
    rows are fp64 softmaxes (draft_attention_rows, src/toymodel.py:315-352),
    summed over the rows on the committed positions, reduced over the head
    group, selected with the reference rule.  Returns the mean recall
    |S_dev ∩ S_ref| / |S_ref| and Jaccard over the committed selections
    (the in-block tail is common to both) and the count of identical masks.

    draft_q [B, Ld, Hqd, R, dd], draft_k [B, Ld, Hkvd, N, dd] (device)."""
    import torch

    s = step.shape
    cfg = cfg if cfg is not None else step.cfg
    R, base = s.rows, s.context
    nd = s.draft_layers * s.draft_q_heads
    Gd = s.draft_group
    src = step.row_src.cpu().numpy()
    idx = step.idx.index_select(0, torch.tensor(units, device=step.idx.device)).cpu().numpy()
    cnt = step.cnt.index_select(0, torch.tensor(units, device=step.cnt.device)).cpu().numpy()
    rec, jac, same = [], [], 0
    cache = {}
    for j, u in enumerate(units):
        rows = []
        for hj in src[u]:
            hj = int(hj)
            if hj not in cache:
                b, rest = divmod(hj, nd)
                dl, dh = divmod(rest, s.draft_q_heads)
                q = draft_q[b, dl, dh].float().cpu().numpy()                       # [R, dd]
                keys = draft_k[b, dl, dh // Gd, : base + R].float().cpu().numpy()   # [n_kv, dd]
                p = O.draft_attention_rows(q, keys, base, R)
                cache[hj] = O.reduce_rows_fp32([x[:base] for x in p])              # committed positions
            rows.append(cache[hj])
        red = O.reduce_rows_fp32(rows)
        ref = O.select_committed(red, base, int(step.budget), oracle_config(cfg))
        dev = idx[j, : cnt[j]].astype(np.int64)
        dev = dev[dev < base]
        inter = np.intersect1d(dev, ref).size
        rec.append(inter / max(1, ref.size))
        jac.append(inter / max(1, np.union1d(dev, ref).size))
        same += int(np.array_equal(dev, ref))
    return {"units": len(units), "recall": round(float(np.mean(rec)), 5), "jaccard": round(float(np.mean(jac)), 5),
            "identical_masks": same, "min_recall": round(float(np.min(rec)), 5),
            "what": "device masks (bf16 capture -> fp32 rows -> select) vs masks from fp64 reference draft rows "
                    "on the same bf16 inputs, committed positions"}
