"""Model-level drop-in and the device-resident verify loop vs the reference.

* ``forward_prefill / forward_block / forward_decode / replay_position`` with
  masks, ``record_attention`` and ``record_scores`` (src/toymodel.py:359-455)
  against ``tests/golden/forward_records.npz`` (reference outputs).
* ``specdec.generate`` (src/specdec.py:258-383) — tokens, statistics,
  per-round outcomes, the exact event log and mask dump — and
  ``greedy_generate`` against ``tests/golden/generate/*.json``, produced by
  the reference itself (tests/golden/make_generate_golden.py), including
  BASELINE config 1 (draft 2L/4H, target 4L/8H, d 64, 4K context, 90%
  sparsity, gamma 4).
* The reference's OWN ``specdec.generate`` (from baseline/_ref) with the
  INTEGRATION.md seam applied — its forwards and mask functions replaced by
  this package's — reproduces the same golden runs.
"""

from __future__ import annotations

import hashlib
import io
import json
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import sts_oracle as O

ROOT = Path(__file__).resolve().parent.parent
GOLD = ROOT / "tests" / "golden"
CASES = sorted(p.stem for p in (GOLD / "generate").glob("*.json"))
REF = ROOT / "baseline" / "_ref"

pytestmark = pytest.mark.gpu


def _doc(name):
    return json.loads((GOLD / "generate" / f"{name}.json").read_text())


def _weights(cfg):
    return O.init_model(O.OracleModelConfig(**cfg))


def _pair(doc):
    target = _weights(doc["target_config"])
    draft = target if doc["draft_config"] is None else _weights(doc["draft_config"])
    return draft, target


def _mappings(doc, tmp_path, load_mapping, MappingSet):
    paths = []
    for i, m in enumerate(doc["mappings"]):
        p = tmp_path / f"map{i}.json"
        p.write_text(json.dumps(m))
        paths.append(p)
    return MappingSet.from_paths(paths) if paths else None


def _sha(s: str) -> str:
    return hashlib.sha256(s.encode()).hexdigest()


def _check_result(res, log, dump, exp):
    assert res.tokens == exp["tokens"]
    assert res.new_tokens == exp["new_tokens"]
    assert res.stats.to_dict() == exp["stats"]
    assert [[r.proposed, r.accepted_len, r.correction_token, r.masks_used] for r in res.rounds] == exp["rounds"]
    if exp["event_log"]["text"] is not None:
        assert log == exp["event_log"]["text"]
    assert _sha(log) == exp["event_log"]["sha256"]
    assert _sha(dump) == exp["mask_dump"]["sha256"], "mask dump differs from the reference's"


# -- forwards ------------------------------------------------------------------------


def test_forwards_match_reference_records():
    import torch

    import paper_2605_15508_b200 as P

    g = np.load(GOLD / "forward_records.npz")
    cfg = dict(layers=2, heads=3, head_dim=8, vocab=32, max_seq=64, page_size=4, seed=5)
    w = _weights(cfg)

    def check(tag, rec, logits_key):
        np.testing.assert_allclose(rec.logits, g[logits_key], rtol=1e-5, atol=1e-6)
        for l in range(2):
            for h in range(3):
                a, s = rec.attention[(l, h)], rec.scores[(l, h)]
                assert a.dtype == np.float32 and a.shape == g[f"{tag}_att_{l}_{h}"].shape
                np.testing.assert_allclose(a, g[f"{tag}_att_{l}_{h}"], rtol=1e-6, atol=1e-7)
                np.testing.assert_allclose(s, g[f"{tag}_sc_{l}_{h}"], rtol=1e-6, atol=1e-6)
                # zeros outside the allowed set / beyond the causal prefix are exact
                assert np.array_equal(a == 0, g[f"{tag}_att_{l}_{h}"] == 0)

    rec, cache = P.forward_prefill(w, g["prefill_tokens"].tolist(), record_attention=True, record_scores=True)
    assert isinstance(cache, P.PagedKVCache) and cache.length == 20
    check("prefill", rec, "prefill_logits")
    masks = {key: [g[f"block_mask_{key[0]}_{key[1]}_{r}"] for r in range(4)] for key in ((0, 0), (1, 2))}
    rec = P.forward_block(w, g["block_tokens"].tolist(), cache, masks=masks, record_attention=True,
                          record_scores=True)
    check("block", rec, "block_logits")
    dmask = {(0, 1): g["decode_mask_0_1"], (1, 0): g["decode_mask_1_0"]}
    rec = P.forward_decode(w, int(g["decode_token"][0]), cache, masks=dmask, record_attention=True,
                           record_scores=True)
    check("decode", rec, "decode_logits")
    r = P.replay_position(w, cache, 10, int(g["prefill_tokens"][10]), masks={(0, 2): np.array([0, 4, 9])})
    np.testing.assert_allclose(r, g["replay_logits"], rtol=1e-5, atol=1e-6)
    # reference contract errors
    with pytest.raises(P.ContractViolation, match="escapes the causal prefix"):
        P.forward_block(w, [1, 2], cache, masks={(0, 0): [np.array([0]), np.array([10_000])]})
    with pytest.raises(P.ContractViolation, match="empty mask row"):
        P.forward_block(w, [1], cache, masks={(0, 0): [np.array([], dtype=np.int64)]})
    with pytest.raises(P.ContractViolation, match="covers 1 rows"):
        P.forward_block(w, [1, 2], cache, masks={(0, 0): [np.array([0])]})
    with pytest.raises(P.InputError):
        P.forward_decode(w, 99, cache)
    torch.cuda.synchronize()


# -- the integrated loop -----------------------------------------------------------


@pytest.mark.parametrize("name", CASES)
def test_generate_matches_reference(name, tmp_path):
    import paper_2605_15508_b200 as P

    doc = _doc(name)
    draft, target = _pair(doc)
    mappings = _mappings(doc, tmp_path, P.load_mapping, P.MappingSet)
    sparsity = P.SparsityConfig(**doc["sparsity"]) if doc["sparsity"] is not None else None
    cfg = P.SpecConfig(gamma=doc["gamma"], sparsity=sparsity, mappings=mappings)
    log, dump = io.StringIO(), io.StringIO()
    res = P.generate(draft, target, doc["prompt"], doc["max_new"], cfg, event_log=log, mask_dump=dump)
    _check_result(res, log.getvalue(), dump.getvalue(), doc["expected"])
    assert P.greedy_generate(target, doc["prompt"], doc["max_new"]) == doc["expected"]["greedy_tokens"]


def test_generate_single_stream_equals_overlapped(tmp_path):
    import paper_2605_15508_b200 as P

    doc = _doc("self_sparse")
    draft, target = _pair(doc)
    mappings = _mappings(doc, tmp_path, P.load_mapping, P.MappingSet)
    cfg = P.SpecConfig(gamma=doc["gamma"], sparsity=P.SparsityConfig(**doc["sparsity"]), mappings=mappings)
    a = P.generate(draft, target, doc["prompt"], doc["max_new"], cfg, overlap=False)
    b = P.generate(draft, target, doc["prompt"], doc["max_new"], cfg, overlap=True)
    assert a.tokens == b.tokens == doc["expected"]["tokens"]


def test_propose_verify_reference_named(tmp_path):
    """propose / verify / ModelSession (src/specdec.py:100-209) on the golden
    self-speculation case: the first round's outcome."""
    import paper_2605_15508_b200 as P

    doc = _doc("small_dense_spec")
    draft_w, target_w = _pair(doc)
    draft, target = P.ModelSession(draft_w), P.ModelSession(target_w)
    draft.prefill(doc["prompt"])
    target.prefill(doc["prompt"])
    tokens, rows = P.propose(draft, doc["gamma"])
    assert len(rows) == doc["gamma"] and all(len(r) == draft_w.config.layers * draft_w.config.heads for r in rows)
    assert rows[0][(0, 0)].shape == (len(doc["prompt"]) + 1,)
    out = P.verify(target, tokens, None)
    first = doc["expected"]["rounds"][0]
    assert [out.proposed, out.accepted_len, out.correction_token, out.masks_used] == first
    assert target.length == len(doc["prompt"]) + out.accepted_len
    with pytest.raises(P.ContractViolation, match="cover"):
        P.verify(target, [1, 2], {(0, 0): [np.array([0])] * 2})


# -- the reference's own loop through the INTEGRATION.md seam ------------------------


def _ref_modules():
    if not (REF / "specsparse").is_dir():
        pytest.skip("baseline/_ref (the installed reference, INTEGRATION.md) is not present on this box")
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import specsparse.headmap as RH
    import specsparse.sparsity as RSP
    import specsparse.specdec as RS
    import specsparse.toymodel as RT

    return RS, RT, RH, RSP


@pytest.mark.parametrize("name", ["small_token", "small_prefill_decode", "small_int_budget_nocurrent",
                                  "self_pages", "c1"])
def test_reference_generate_through_seam(name, tmp_path, monkeypatch):
    import paper_2605_15508_b200 as P

    RS, RT, RH, RSP = _ref_modules()
    for attr, fn in (("forward_prefill", P.forward_prefill), ("forward_decode", P.forward_decode),
                     ("forward_block", P.forward_block), ("draft_masks_decode", P.draft_masks_decode),
                     ("draft_masks_prefill", P.draft_masks_prefill), ("remap_masks", P.remap_masks),
                     ("_verification_masks", P.verification_masks)):
        monkeypatch.setattr(RS, attr, fn)
    doc = _doc(name)
    target = RT.init_model(RT.ModelConfig(**doc["target_config"]))
    draft = target if doc["draft_config"] is None else RT.init_model(RT.ModelConfig(**doc["draft_config"]))
    mappings = _mappings(doc, tmp_path, RH.load_mapping, RH.MappingSet)
    cfg = RS.SpecConfig(gamma=doc["gamma"], sparsity=RSP.SparsityConfig(**doc["sparsity"]), mappings=mappings)
    log, dump = io.StringIO(), io.StringIO()
    res = RS.generate(draft, target, doc["prompt"], doc["max_new"], cfg, event_log=log, mask_dump=dump)
    _check_result(res, log.getvalue(), dump.getvalue(), doc["expected"])
