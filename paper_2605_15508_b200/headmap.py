"""Head-mapping tables consumed by the hot path (src/headmap.py:30-56, :170-186).

The runtime side: ``HeadMapping.entries`` (target head -> (draft head,
score)) and ``MappingSet.nearest``; ``to_table`` lowers a mapping to the int32
indirection table the kernels use instead of copying masks per target head.
The offline search ``find_head_mapping`` (Algorithm 1) runs
on the GPU: per-row top-k sets from the radix select, bitsets, and a popcount
overlap kernel (include/sts_b200.h sts_topk_bitsets / sts_bitset_overlap).
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .errors import ContractViolation, InputError

HeadKey = tuple[int, int]  # (layer, head), src/toymodel.py:28


@dataclass
class HeadMapping:
    """Per-k table pairing each target head with one draft head (src/headmap.py:30-44)."""

    k: int
    entries: dict  # HeadKey -> (HeadKey, score)
    trace_set_id: str = ""
    draft_config: object = None
    target_config: object = None

    def draft_for(self, target: HeadKey) -> HeadKey:
        try:
            return self.entries[target][0]
        except KeyError:
            raise ContractViolation(f"mapping has no entry for target head {target}") from None

    def layer_distance_stats(self) -> dict:
        """Distribution of |target layer - draft layer| (src/headmap.py:46-56)."""
        dists = [abs(t[0] - d[0]) for t, (d, _) in self.entries.items()]
        hist: dict = {}
        for v in sorted(dists):
            hist[str(v)] = hist.get(str(v), 0) + 1
        return {"mean": float(np.mean(dists)), "max": int(max(dists)), "histogram": hist}

    def to_table(self, target_layers: int, target_heads: int, draft_heads: int) -> np.ndarray:
        """int32 [target_layers, target_heads] of flattened draft (layer*H_d + head)."""
        table = np.empty((target_layers, target_heads), dtype=np.int32)
        for tl in range(target_layers):
            for th in range(target_heads):
                dl, dh = self.draft_for((tl, th))
                if not 0 <= dh < draft_heads:
                    raise ContractViolation(f"draft head {(dl, dh)} outside {draft_heads} heads")
                table[tl, th] = dl * draft_heads + dh
        return table

    @classmethod
    def from_table(cls, k: int, table) -> "HeadMapping":
        table = np.asarray(table)
        raise_if = table.ndim != 3 or table.shape[-1] != 2
        if raise_if:
            raise InputError("table must be [target_layers, target_heads, 2] of (draft layer, head)")
        entries = {
            (tl, th): ((int(table[tl, th, 0]), int(table[tl, th, 1])), 0)
            for tl in range(table.shape[0])
            for th in range(table.shape[1])
        }
        return cls(k, entries, "table")


class MappingSet:
    """All stored mappings; ``nearest`` picks per round (src/headmap.py:170-186)."""

    def __init__(self, mappings):
        if not mappings:
            raise InputError("MappingSet needs at least one mapping")
        self.mappings = sorted(mappings, key=lambda m: m.k)

    def nearest(self, budget: int) -> HeadMapping:
        return min(self.mappings, key=lambda m: (abs(m.k - budget), m.k))

    @classmethod
    def from_paths(cls, paths) -> "MappingSet":
        """src/headmap.py:184-186."""
        return cls([load_mapping(p) for p in paths])


MAPPING_FORMAT_VERSION = 1


def _config_dict(cfg) -> dict:
    if hasattr(cfg, "to_dict"):
        return cfg.to_dict()
    return dict(cfg)


def save_mapping(mapping: HeadMapping, path) -> None:
    """Write a mapping as versioned JSON with layer-distance statistics
    (src/headmap.py:128-143; byte-identical documents)."""
    doc = {
        "format_version": MAPPING_FORMAT_VERSION,
        "k": mapping.k,
        "trace_set_id": mapping.trace_set_id,
        "draft_config": _config_dict(mapping.draft_config),
        "target_config": _config_dict(mapping.target_config),
        "entries": [[t[0], t[1], d[0], d[1], score] for t, (d, score) in sorted(mapping.entries.items())],
        "layer_distance": mapping.layer_distance_stats(),
    }
    Path(path).write_text(json.dumps(doc, indent=2, sort_keys=True))


def load_mapping(path) -> HeadMapping:
    """Read the reference's mapping JSON (src/headmap.py:146-165): format_version
    1, ``entries`` = [[target_layer, target_head, draft_layer, draft_head, score]],
    model configs as ``ModelConfig``."""
    path = Path(path)
    try:
        doc = json.loads(path.read_text())
    except (OSError, json.JSONDecodeError) as exc:
        raise InputError(f"cannot read mapping {path}: {exc}") from exc
    if doc.get("format_version") != MAPPING_FORMAT_VERSION:
        raise InputError(f"unsupported mapping format version {doc.get('format_version')!r} in {path}")
    try:
        entries = {(int(tl), int(th)): ((int(dl), int(dh)), int(score)) for tl, th, dl, dh, score in doc["entries"]}
    except (KeyError, TypeError, ValueError) as exc:
        raise InputError(f"bad mapping file {path}: {exc}") from exc
    from .model import ModelConfig

    return HeadMapping(k=int(doc["k"]), entries=entries, trace_set_id=str(doc["trace_set_id"]),
                       draft_config=ModelConfig.from_dict(doc["draft_config"]),
                       target_config=ModelConfig.from_dict(doc["target_config"]))


def find_head_mapping(ts, k: int) -> HeadMapping:
    """Best-overlap draft head for every target head (src/headmap.py:83-125),
    on the GPU.

    ``ts``: a trace set (the reference's ``TraceSet`` or any object with
    ``samples`` — each with ``draft`` / ``target`` dicts of causal attention
    matrices [n, n] keyed (layer, head) — and ``draft_config`` /
    ``target_config`` with ``layers`` and ``heads``).  Per sample and head,
    row t's set is the top-k of its prefix [0, t] (``rowwise_topk_sets``, the
    tie rule of topk_indices); score(th, dh) = sum over samples and rows of
    |set_th(t) & set_dh(t)|; ties go to the smallest (layer, head).
    """
    import torch

    from . import _lib, kernels
    from ._lib import call, ptr, stream_handle

    if k < 1:
        raise ContractViolation(f"k must be >= 1, got {k}")
    if not ts.samples:
        raise InputError("cannot build a mapping from an empty trace set")
    draft_heads = [(l, h) for l in range(ts.draft_config.layers) for h in range(ts.draft_config.heads)]
    target_heads = [(l, h) for l in range(ts.target_config.layers) for h in range(ts.target_config.heads)]
    if not torch.cuda.is_available():
        raise RuntimeError("find_head_mapping runs on the GPU (there is no CPU fallback)")
    dev = torch.device("cuda", torch.cuda.current_device())
    scores = torch.zeros((len(target_heads), len(draft_heads)), dtype=torch.int64, device=dev)

    def bitsets(mats, heads, n, words):
        rows = torch.stack([torch.as_tensor(np.asarray(mats[hk], dtype=np.float32)) for hk in heads]).to(dev)
        rows = rows.reshape(len(heads) * n, n)
        if n % 4:
            rows = torch.nn.functional.pad(rows, (0, 4 - n % 4))
        row_len = torch.arange(1, n + 1, dtype=torch.int32, device=dev).repeat(len(heads))
        idx, cnt = kernels.select_topk(rows.contiguous(), row_len=row_len, budget=int(k), include_current=False)
        bits = torch.empty((len(heads) * n, words), dtype=torch.int32, device=dev)
        call("sts_topk_bitsets", ptr(idx), idx.stride(0), ptr(cnt), len(heads) * n, words, ptr(bits),
             stream_handle())
        return bits.reshape(len(heads), n * words)

    for sample in ts.samples:
        n = int(sample.length)
        words = -(-n // 32)
        words = -(-words // 4) * 4  # 16-byte rows for the vector loads
        tb = bitsets(sample.target, target_heads, n, words)
        db = bitsets(sample.draft, draft_heads, n, words)
        call("sts_bitset_overlap", ptr(tb), len(target_heads), ptr(db), len(draft_heads), n * words, ptr(scores),
             stream_handle())
    totals = scores.cpu().numpy()
    entries = {}
    for i, th in enumerate(target_heads):
        best = int(np.argmax(totals[i]))  # first max = lexicographically smallest draft head
        entries[th] = (draft_heads[best], int(totals[i, best]))
    cid = ts.content_id() if hasattr(ts, "content_id") else ""
    return HeadMapping(k=k, entries=entries, trace_set_id=cid, draft_config=ts.draft_config,
                       target_config=ts.target_config)
