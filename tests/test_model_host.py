"""Host-side logic of the model-level drop-in (no GPU): mapping I/O against
the reference's own documents, ModelConfig, duck-typed sparsity configs."""

from __future__ import annotations

import json
from pathlib import Path
from types import SimpleNamespace

import pytest

import paper_2605_15508_b200 as P
from paper_2605_15508_b200.sparsity import select_kwargs
from paper_2605_15508_b200.specdec import _tokens_for_context, _touched_pages

GOLD = Path(__file__).resolve().parent / "golden" / "generate"


def _mapping_docs():
    for p in sorted(GOLD.glob("*.json")):
        for m in json.loads(p.read_text())["mappings"]:
            yield p.stem, m


def test_mapping_roundtrip_is_byte_identical(tmp_path):
    """load_mapping -> save_mapping reproduces the reference's save_mapping
    document (src/headmap.py:128-165), layer-distance stats included."""
    n = 0
    for name, doc in _mapping_docs():
        src = tmp_path / f"{name}_{doc['k']}.json"
        src.write_text(json.dumps(doc, indent=2, sort_keys=True))
        m = P.load_mapping(src)
        assert isinstance(m.draft_config, P.ModelConfig) and isinstance(m.target_config, P.ModelConfig)
        assert m.layer_distance_stats() == doc["layer_distance"]
        out = tmp_path / "out.json"
        P.save_mapping(m, out)
        assert out.read_text() == src.read_text()
        n += 1
    assert n >= 10


def test_mapping_set_from_paths_nearest(tmp_path):
    doc = json.loads((GOLD / "c1.json").read_text())
    paths = []
    for m in doc["mappings"]:
        p = tmp_path / f"k{m['k']}.json"
        p.write_text(json.dumps(m))
        paths.append(p)
    ms = P.MappingSet.from_paths(paths)
    assert [m.k for m in ms.mappings] == sorted(m["k"] for m in doc["mappings"])
    assert ms.nearest(401).k == 400 and ms.nearest(73).k == 128 and ms.nearest(72).k == 16  # tie -> smaller k
    with pytest.raises(P.InputError):
        P.load_mapping(tmp_path / "missing.json")


def test_model_config_contract():
    c = P.ModelConfig.from_dict({"layers": 2, "heads": 4, "head_dim": 8, "vocab": 16, "max_seq": 32})
    assert c.hidden == 32 and c.to_dict()["page_size"] == 4
    with pytest.raises(P.ConfigError):
        P.ModelConfig(layers=0, heads=1, head_dim=1, vocab=1, max_seq=1)
    with pytest.raises(P.InputError):
        P.ModelConfig.from_dict({"layers": "x"})


def test_duck_typed_sparsity_config():
    """The reference's own SparsityConfig (any object with its fields) drives
    the drop-in functions (INTEGRATION.md seam)."""
    ref_like = SimpleNamespace(budget=0.1, page_size=4, include_current=False, include_sink=True, recent_window=2,
                               scope="decode")
    kw = select_kwargs(ref_like)
    assert kw == dict(budget=0.1, page_size=4, include_current=False, include_sink=True, recent_window=2)
    assert _tokens_for_context(ref_like, 4000) == 400 and _tokens_for_context(SimpleNamespace(budget=7), 9) == 7


def test_touched_pages_wire_format():
    cfg = SimpleNamespace(page_size=4, layers=2, heads=2)
    dense = _touched_pages(9, cfg, None)
    assert dense[0] == [[h, p] for h in range(2) for p in range(3)]
    import numpy as np

    sparse = _touched_pages(9, cfg, [{(0, 1): [np.array([0, 5])], (1, 0): np.array([8])}, None][:1])
    assert sparse == [[[1, 0], [1, 1]], [[0, 2]]]
