"""Generate golden vectors by running the REAL reference package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``specsparse`` from /root/reference/pkg/src (read-only), runs the
hot-path functions on seeded inputs and writes ``tests/golden/*.npz``. The
fixtures are committed; nothing on the GPU box reads /root/reference.

Functions exercised (reference file:line):
  numkit.topk_indices            src/numkit.py:74-86
  sparsity.page_aggregate        src/sparsity.py:72-83
  sparsity.draft_masks_decode    src/sparsity.py:115-119 (-> _select_row :86-112)
  sparsity.draft_masks_prefill   src/sparsity.py:122-130
  sparsity.remap_masks           src/sparsity.py:133-149
  specdec._verification_masks    src/specdec.py:219-233
  sparsity.sparse_attention      src/sparsity.py:152-173
  toymodel forward_decode(record_attention=True) -> ForwardRecord.attention
                                 src/toymodel.py:315-352, :402-427
"""

from __future__ import annotations

import json
import math
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def _pack(arrs, dtype):
    arrs = [np.asarray(a, dtype=dtype).ravel() for a in arrs]
    offs = np.zeros(len(arrs) + 1, dtype=np.int64)
    offs[1:] = np.cumsum([a.size for a in arrs])
    data = np.concatenate(arrs) if arrs else np.zeros(0, dtype)
    return data, offs


def _row_kinds(rng, n, kind):
    if kind == "softmax":
        z = 2.0 * rng.standard_normal(n)
        w = np.exp(z - z.max())
        return (w / w.sum()).astype(np.float32)
    if kind == "ties":
        z = 2.0 * rng.standard_normal(n)
        w = np.exp(z - z.max())
        w = (w / w.sum()).astype(np.float32)
        return (np.round(w * 256.0) / 256.0).astype(np.float32)  # quantised to 2^-8
    if kind == "special":
        x = rng.standard_normal(n).astype(np.float32)
        m = rng.random(n)
        x[m < 0.05] = np.nan
        x[(m >= 0.05) & (m < 0.08)] = -0.0
        x[(m >= 0.08) & (m < 0.11)] = 0.0
        x[(m >= 0.11) & (m < 0.13)] = np.inf
        x[(m >= 0.13) & (m < 0.15)] = -np.inf
        return x
    if kind == "uniform":
        return np.full(n, 1.0 / n, dtype=np.float32)
    raise ValueError(kind)


def main() -> None:
    sys.path.insert(0, str(REF))
    import specsparse  # noqa: F401
    from specsparse import numkit, sparsity, specdec
    from specsparse.headmap import HeadMapping
    from specsparse.toymodel import ModelConfig

    rng = np.random.default_rng(20260517)

    # ---- 1. topk_indices -------------------------------------------------
    rows, ks, outs = [], [], []
    for kind in ("softmax", "ties", "special", "uniform"):
        for n in (1, 2, 3, 7, 31, 64, 257, 1000, 4097):
            for k in sorted({1, 2, max(1, n // 10), max(1, n // 2), n - 1 if n > 1 else 1, n, n + 5}):
                r = _row_kinds(rng, n, kind)
                rows.append(r)
                ks.append(k)
                outs.append(numkit.topk_indices(r, k))
    rd, ro = _pack(rows, np.float32)
    od, oo = _pack(outs, np.int64)
    np.savez_compressed(OUT / "topk.npz", rows=rd, row_offs=ro, k=np.asarray(ks), out=od, out_offs=oo)

    # ---- 2. page_aggregate -------------------------------------------------
    rows, ps_list, outs = [], [], []
    for n in (1, 5, 16, 17, 100, 333, 1000, 4097):
        for ps in (1, 2, 3, 7, 8, 9, 15, 16, 17, 31, 32, 64, 127, 128, 129, 200, 300):
            r = _row_kinds(rng, n, "softmax") * np.float32(rng.uniform(0.5, 50))
            rows.append(r)
            ps_list.append(ps)
            outs.append(sparsity.page_aggregate(r, ps))
    rd, ro = _pack(rows, np.float32)
    od, oo = _pack(outs, np.float64)
    np.savez_compressed(OUT / "page_aggregate.npz", rows=rd, row_offs=ro, page_size=np.asarray(ps_list), out=od, out_offs=oo)

    # ---- 3. draft_masks_decode / _select_row ------------------------------
    cfg_specs = []
    for budget in (1, 2, 5, 40, 410, 0.1, 0.02, 0.5, 1.0, 1 / 8):
        for ps in (1, 2, 4, 16):
            for cur, sink, win in ((True, False, 0), (False, False, 0), (True, True, 16), (False, True, 3)):
                cfg_specs.append((budget, ps, cur, sink, win))
    rows, cfgs, outs = [], [], []
    for ci, (budget, ps, cur, sink, win) in enumerate(cfg_specs):
        cfg = sparsity.SparsityConfig(budget=budget, page_size=ps, include_current=cur, include_sink=sink, recent_window=win)
        for kind in ("softmax", "ties", "special"):
            n = int(rng.choice([1, 2, 9, 64, 100, 513, 4097]))
            r = _row_kinds(rng, n, kind)
            m = sparsity.draft_masks_decode({(0, 0): r}, cfg)[(0, 0)]
            rows.append(r)
            cfgs.append([budget, isinstance(budget, int), ps, cur, sink, win])
            outs.append(m)
    rd, ro = _pack(rows, np.float32)
    od, oo = _pack(outs, np.int64)
    np.savez_compressed(OUT / "select_row.npz", rows=rd, row_offs=ro, cfg=json.dumps(cfgs), out=od, out_offs=oo)

    # ---- 4. verification masks at the config-1 shape -----------------------
    # draft 2L/4H, target 4L/8H, gamma=4, base=4096, 90% sparsity (budget 0.1)
    dcfg = ModelConfig(layers=2, heads=4, head_dim=64, vocab=64, max_seq=8192, seed=1)
    tcfg = ModelConfig(layers=4, heads=8, head_dim=64, vocab=64, max_seq=8192, seed=2)
    draft_heads = [(l, h) for l in range(2) for h in range(4)]
    entries = {
        (l, h): (draft_heads[int(rng.integers(0, len(draft_heads)))], 0)
        for l in range(4)
        for h in range(8)
    }
    mapping = HeadMapping(410, entries, "golden", dcfg, tcfg)
    vm = {}
    for variant, kind, cfg in (
        ("token", "softmax", sparsity.SparsityConfig(budget=0.1)),
        ("ties", "ties", sparsity.SparsityConfig(budget=0.1)),
        ("page16", "softmax", sparsity.SparsityConfig(budget=0.1, page_size=16)),
        ("extras", "softmax", sparsity.SparsityConfig(budget=0.1, include_sink=True, recent_window=64)),
    ):
        base, gamma = 4096, 4
        draft_rows = [
            {hd: _row_kinds(rng, base + i + 1, kind) for hd in draft_heads} for i in range(gamma)
        ]
        masks = specdec._verification_masks(draft_rows, base, cfg, mapping)
        vm[f"{variant}_rows"] = np.stack(
            [np.stack([np.pad(draft_rows[i][hd], (0, gamma - 1 - i)) for hd in draft_heads]) for i in range(gamma)]
        )  # (gamma, 8 draft heads, base+gamma) zero-padded
        tgt_keys = sorted(masks)
        data, offs = _pack([masks[t][i] for t in tgt_keys for i in range(gamma)], np.int64)
        vm[f"{variant}_out"] = data
        vm[f"{variant}_offs"] = offs
        vm[f"{variant}_cfg"] = json.dumps([cfg.budget, cfg.page_size, cfg.include_current, cfg.include_sink, cfg.recent_window])
    vm["entries"] = np.asarray([[t[0], t[1], d[0], d[1]] for t, (d, _) in sorted(entries.items())], dtype=np.int64)
    vm["draft_heads"] = np.asarray(draft_heads, dtype=np.int64)
    np.savez_compressed(OUT / "verification_c1.npz", **vm)

    # ---- 5. prefill masks ----------------------------------------------------
    pm = {}
    mats = []
    outs = []
    cfgs = []
    for n, budget, ps in ((5, 2, 1), (12, 3, 2), (33, 0.25, 1), (40, 0.1, 4), (64, 8, 1)):
        mat = numkit.row_softmax(rng.standard_normal((n, n)), range(1, n + 1))
        cfg = sparsity.SparsityConfig(budget=budget, page_size=ps)
        got = sparsity.draft_masks_prefill({(0, 0): mat}, cfg)[(0, 0)]
        mats.append(mat)
        outs.extend(got)
        cfgs.append([n, budget, ps])
    md, mo = _pack(mats, np.float32)
    od, oo = _pack(outs, np.int64)
    np.savez_compressed(OUT / "prefill.npz", mats=md, mat_offs=mo, cfg=json.dumps(cfgs), out=od, out_offs=oo)

    # ---- 6. sparse_attention -----------------------------------------------
    qs, ks_, vs, masks, outs, shapes = [], [], [], [], [], []
    for case in range(24):
        n = int(rng.integers(1, 300))
        d = int(rng.choice([4, 8, 64, 128]))
        q = rng.standard_normal(d).astype(np.float32)
        k = rng.standard_normal((n, d)).astype(np.float32)
        v = rng.standard_normal((n, d)).astype(np.float32)
        size = int(rng.integers(1, n + 1))
        mask = np.sort(rng.choice(n, size=size, replace=False))
        out = sparsity.sparse_attention(q, k, v, mask)
        qs.append(q); ks_.append(k); vs.append(v); masks.append(mask); outs.append(out); shapes.append([n, d])
    np.savez_compressed(
        OUT / "sparse_attention.npz",
        q=_pack(qs, np.float32)[0], k=_pack(ks_, np.float32)[0], v=_pack(vs, np.float32)[0],
        mask=_pack(masks, np.int64)[0], mask_offs=_pack(masks, np.int64)[1],
        out=_pack(outs, np.float32)[0], shapes=np.asarray(shapes, dtype=np.int64),
    )

    # ---- 7. draft score capture through the toy model ------------------------
    # Layer-0 queries are recomputed with the reference's own helpers
    # (toymodel._rms_norm, numkit.matmul; src/toymodel.py:307,316-317) so the
    # oracle's draft_attention_rows can be pinned against ForwardRecord.attention.
    from specsparse import toymodel
    from specsparse.toymodel import forward_decode, forward_prefill, init_model

    cfg = ModelConfig(layers=2, heads=4, head_dim=16, vocab=64, max_seq=256, seed=11)
    w = init_model(cfg)
    toks = rng.integers(0, 64, size=120)
    _, cache = forward_prefill(w, toks[:100])
    rows, qs = [], []
    for i, t in enumerate(toks[100:104]):
        pos = cache.length
        rec = forward_decode(w, int(t), cache, record_attention=True)
        x = w.token_emb[[int(t)]] + w.pos_emb[pos : pos + 1]
        h = toymodel._rms_norm(x, w.attn_norm[0])
        q = numkit.matmul(h, w.wq[0]).reshape(cfg.heads, cfg.head_dim)
        qs.append(q)
        rows.append(np.stack([np.pad(rec.attention[(0, hh)][0], (0, 3 - i)) for hh in range(cfg.heads)]))
    np.savez_compressed(
        OUT / "capture.npz",
        keys0=cache.keys(0),  # (104, H, d) layer-0 keys
        q0=np.stack(qs),  # (4 steps, H, d)
        rows=np.stack(rows),  # (4 steps, H, 104) zero-padded
        base=np.asarray(100),
    )
    make_headmap_golden()
    print("golden vectors written to", OUT)


def make_headmap_golden():
    """Algorithm 1 (headmap.find_head_mapping, src/headmap.py:83-125) on
    synthetic paired traces: 2 samples, draft 2L x 3H, target 2L x 4H, for
    k in (1, 3, 8); softmax rows plus tie-heavy rows."""
    sys.path.insert(0, str(REF))
    from specsparse import headmap, numkit
    from specsparse.toymodel import ModelConfig
    from specsparse.tracestore import TraceSample, TraceSet

    rng = np.random.default_rng(77)
    dcfg = ModelConfig(layers=2, heads=3, head_dim=8, vocab=32, max_seq=64)
    tcfg = ModelConfig(layers=2, heads=4, head_dim=8, vocab=32, max_seq=64)
    samples, mats = [], {}
    for si, n in enumerate((23, 40)):
        def mat(tie):
            z = rng.standard_normal((n, n)) * 2.0
            m = numkit.row_softmax(z, range(1, n + 1)).astype(np.float32)
            if tie:
                m = (np.round(m * 16) / 16).astype(np.float32)
            return m
        draft = {(l, h): mat(h == 2) for l in range(2) for h in range(3)}
        target = {(l, h): mat(h == 3) for l in range(2) for h in range(4)}
        samples.append(TraceSample(length=n, draft=draft, target=target))
        for key, m in draft.items():
            mats[f"s{si}_d{key[0]}_{key[1]}"] = m
        for key, m in target.items():
            mats[f"s{si}_t{key[0]}_{key[1]}"] = m
    ts = TraceSet(draft_config=dcfg, target_config=tcfg, samples=samples)
    res = {}
    for k in (1, 3, 8):
        mp = headmap.find_head_mapping(ts, k)
        res[str(k)] = [[tl, th, mp.entries[(tl, th)][0][0], mp.entries[(tl, th)][0][1], int(mp.entries[(tl, th)][1])]
                       for tl in range(2) for th in range(4)]
    np.savez_compressed(OUT / "headmap.npz", result=json.dumps(res), lengths=np.asarray([23, 40]), **mats)


if __name__ == "__main__":
    main()
