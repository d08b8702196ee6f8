"""Head-mapping tables consumed by the hot path (src/headmap.py:30-56, :170-186).

Only the runtime side is here: ``HeadMapping.entries`` (target head ->
(draft head, score)) and ``MappingSet.nearest``.  The offline search
(find_head_mapping, Algorithm 1) is out of scope ("next").
``to_table`` lowers a mapping to the int32 indirection table the kernels use
instead of copying masks per target head.
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


MAPPING_FORMAT_VERSION = 1


def load_mapping(path) -> HeadMapping:
    """Read the reference's mapping JSON (src/headmap.py:128-165): format_version
    1, ``entries`` = [[target_layer, target_head, draft_layer, draft_head, score]]."""
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
    return HeadMapping(int(doc["k"]), entries, str(doc.get("trace_set_id", "")),
                       doc.get("draft_config"), doc.get("target_config"))
