"""Golden speculative-generation runs of the REAL reference package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_generate_golden.py [--only NAME]

For each case it builds the toy draft/target pair (``init_model``, src/
toymodel.py:126-160), a head-mapping set from traces of a synthetic corpus
(``collect_traces`` + ``find_head_mapping``, src/tracestore.py:68-90,
src/headmap.py:83-125, saved with ``save_mapping`` :128-143), runs
``specdec.generate`` (src/specdec.py:258-383) with ``event_log`` and
``mask_dump`` and ``greedy_generate`` (:386-400), and writes
tests/golden/generate/<case>.json: configs, prompt, mappings, the tokens,
stats, per-round outcomes and the exact event-log / mask-dump text (or its
sha256 when large).  Nothing on the GPU box reads /root/reference.
"""

from __future__ import annotations

import argparse
import hashlib
import io
import json
import sys
import tempfile
import time
from pathlib import Path

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "generate"
INLINE_LIMIT = 200_000

# (name, draft cfg, target cfg, prompt_len, max_new, gamma, sparsity kwargs or None, mapping ks, corpus)
CASES = [
    # BASELINE config 1: draft 2L/4H, target 4L/8H, d_head 64, 4K context, 90% sparsity, gamma 4
    ("c1", dict(layers=2, heads=4, head_dim=64, vocab=256, max_seq=4096, page_size=16, seed=21),
     dict(layers=4, heads=8, head_dim=64, vocab=256, max_seq=4096, page_size=16, seed=22),
     4000, 40, 4, dict(budget=0.1), [16, 128, 400], dict(samples=2, length=64)),
    # the c1 target speculating on itself at 4K: accepted runs under 90% sparsity
    ("c1_self", None, dict(layers=4, heads=8, head_dim=64, vocab=256, max_seq=4096, page_size=16, seed=22),
     4000, 40, 4, dict(budget=0.1), [128, 400], dict(samples=2, length=64)),
    ("small_token", dict(layers=1, heads=2, head_dim=4, vocab=32, max_seq=160, page_size=4, seed=8),
     dict(layers=2, heads=2, head_dim=4, vocab=32, max_seq=160, page_size=4, seed=7),
     48, 24, 4, dict(budget=0.25), [4, 8], dict(samples=4, length=24)),
    ("small_pages_extras", dict(layers=2, heads=2, head_dim=8, vocab=48, max_seq=256, page_size=4, seed=31),
     dict(layers=3, heads=4, head_dim=8, vocab=48, max_seq=256, page_size=4, seed=32),
     120, 30, 3, dict(budget=0.2, page_size=4, include_sink=True, recent_window=3), [8, 24],
     dict(samples=3, length=32)),
    ("small_int_budget_nocurrent", dict(layers=1, heads=4, head_dim=8, vocab=40, max_seq=200, page_size=8, seed=41),
     dict(layers=2, heads=4, head_dim=8, vocab=40, max_seq=200, page_size=8, seed=42),
     90, 20, 5, dict(budget=7, include_current=False), [4, 16], dict(samples=3, length=24)),
    ("small_prefill_decode", dict(layers=2, heads=2, head_dim=8, vocab=32, max_seq=192, page_size=4, seed=51),
     dict(layers=2, heads=4, head_dim=8, vocab=32, max_seq=192, page_size=4, seed=52),
     100, 24, 4, dict(budget=0.3, scope="prefill-decode"), [8, 32], dict(samples=3, length=24)),
    # self-speculation (draft = target weights): long accepted runs, rollbacks at every offset
    ("self_sparse", None, dict(layers=2, heads=4, head_dim=16, vocab=64, max_seq=512, page_size=4, seed=71),
     300, 60, 4, dict(budget=0.5), [64, 150], dict(samples=2, length=40)),
    ("self_pages", None, dict(layers=2, heads=2, head_dim=16, vocab=64, max_seq=512, page_size=8, seed=72),
     200, 60, 6, dict(budget=0.6, page_size=8, include_sink=True), [64, 120], dict(samples=2, length=40)),
    ("small_dense_spec", dict(layers=1, heads=2, head_dim=4, vocab=32, max_seq=96, page_size=4, seed=61),
     dict(layers=2, heads=2, head_dim=4, vocab=32, max_seq=96, page_size=4, seed=62),
     20, 16, 4, None, [], None),
]


def _text(s: str):
    return {"sha256": hashlib.sha256(s.encode()).hexdigest(), "bytes": len(s),
            "text": s if len(s) <= INLINE_LIMIT else None}


def run_case(case):
    from specsparse import numkit
    from specsparse.corpus import synthetic_corpus
    from specsparse.headmap import MappingSet, find_head_mapping, save_mapping
    from specsparse.sparsity import SparsityConfig
    from specsparse.specdec import SpecConfig, generate, greedy_generate
    from specsparse.toymodel import ModelConfig, init_model
    from specsparse.tracestore import collect_traces

    name, dcfg, tcfg, plen, max_new, gamma, skw, ks, corpus_kw = case
    t0 = time.time()
    target = init_model(ModelConfig(**tcfg))
    draft = target if dcfg is None else init_model(ModelConfig(**dcfg))
    prompt = [int(t) for t in numkit.prng_stream(1000 + plen).integers(0, tcfg["vocab"], size=plen)]
    # draft_config None: the draft IS the target (self-speculation)
    mapping_docs = []
    sparsity = None
    mappings = None
    if skw is not None:
        corpus = synthetic_corpus(seed=11, vocab=tcfg["vocab"], **corpus_kw)
        ts = collect_traces(draft, target, corpus)
        maps = [find_head_mapping(ts, k) for k in ks]
        with tempfile.TemporaryDirectory() as td:
            for m in maps:
                p = Path(td) / f"k{m.k}.json"
                save_mapping(m, p)
                mapping_docs.append(json.loads(p.read_text()))
        mappings = MappingSet(maps)
        sparsity = SparsityConfig(**skw)
    cfg = SpecConfig(gamma=gamma, sparsity=sparsity, mappings=mappings)
    log, dump = io.StringIO(), io.StringIO()
    res = generate(draft, target, prompt, max_new, cfg, event_log=log, mask_dump=dump)
    greedy = greedy_generate(target, prompt, max_new)
    doc = {
        "name": name, "draft_config": dcfg, "target_config": tcfg, "prompt": prompt, "max_new": max_new,
        "gamma": gamma, "sparsity": skw, "mappings": mapping_docs,
        "expected": {
            "tokens": res.tokens, "new_tokens": res.new_tokens, "stats": res.stats.to_dict(),
            "rounds": [[r.proposed, r.accepted_len, r.correction_token, r.masks_used] for r in res.rounds],
            "event_log": _text(log.getvalue()), "mask_dump": _text(dump.getvalue()),
            "greedy_tokens": greedy,
        },
        "reference_seconds": round(time.time() - t0, 1),
    }
    OUT.mkdir(exist_ok=True)
    (OUT / f"{name}.json").write_text(json.dumps(doc, sort_keys=True) + "\n")
    print(f"{name}: {len(res.new_tokens)} tokens, {res.stats.rounds} rounds, acceptance "
          f"{res.stats.acceptance_rate:.2f}, {doc['reference_seconds']} s")


FORWARD_CFG = dict(layers=2, heads=3, head_dim=8, vocab=32, max_seq=64, page_size=4, seed=5)


def forward_case():
    """forward_prefill / forward_block / forward_decode / replay_position with
    masks, record_attention and record_scores (src/toymodel.py:359-455) on a
    small model -> tests/golden/forward_records.npz."""
    import numpy as np

    from specsparse import numkit
    from specsparse.toymodel import (ModelConfig, forward_block, forward_decode, forward_prefill, init_model,
                                     replay_position)

    w = init_model(ModelConfig(**FORWARD_CFG))
    rng = numkit.prng_stream(77)
    toks = [int(t) for t in rng.integers(0, 32, size=20)]
    out = {"prefill_tokens": np.array(toks)}
    rec, cache = forward_prefill(w, toks, record_attention=True, record_scores=True)
    out["prefill_logits"] = rec.logits

    def put(tag, r):
        for (l, h), a in r.attention.items():
            out[f"{tag}_att_{l}_{h}"] = a
        for (l, h), a in r.scores.items():
            out[f"{tag}_sc_{l}_{h}"] = a

    put("prefill", rec)
    # masked block of 4 rows: heads (0,0), (1,2) masked per row, the rest dense
    blk = [int(t) for t in rng.integers(0, 32, size=4)]
    base = cache.length
    masks = {}
    for key in ((0, 0), (1, 2)):
        rows = []
        for r in range(4):
            pos = base + r
            sel = np.sort(rng.choice(pos + 1, size=min(pos + 1, 6), replace=False))
            rows.append(sel.astype(np.int64))
            out[f"block_mask_{key[0]}_{key[1]}_{r}"] = rows[-1]
        masks[key] = rows
    out["block_tokens"] = np.array(blk)
    rec = forward_block(w, blk, cache, masks=masks, record_attention=True, record_scores=True)
    out["block_logits"] = rec.logits
    put("block", rec)
    # decode with a decode mask on (0, 1) and (1, 0)
    dmask = {(0, 1): np.array([0, 3, 7], dtype=np.int64), (1, 0): np.array([1, 2, 20], dtype=np.int64)}
    for (l, h), a in dmask.items():
        out[f"decode_mask_{l}_{h}"] = a
    out["decode_token"] = np.array([5])
    rec = forward_decode(w, 5, cache, masks=dmask, record_attention=True, record_scores=True)
    out["decode_logits"] = rec.logits
    put("decode", rec)
    out["replay_logits"] = replay_position(w, cache, 10, toks[10], masks={(0, 2): np.array([0, 4, 9])})
    np.savez_compressed(Path(__file__).resolve().parent / "forward_records.npz", **out)
    print(f"forward_records: {len(out)} arrays")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--only")
    a = ap.parse_args()
    sys.path.insert(0, str(REF))
    if a.only in (None, "forward"):
        forward_case()
    for case in CASES:
        if a.only and case[0] != a.only:
            continue
        run_case(case)
