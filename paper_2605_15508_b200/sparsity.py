"""Reference-named sparsity API, computed on the B200.

Drop-in for ``specsparse.sparsity`` (src/sparsity.py) on the hot path: the
same names, arguments, return types (dicts of int64 numpy index arrays,
fp32 / fp64 numpy results) and exceptions, but every mask / page sum /
attention is produced by libsts_b200.so kernels.  Inputs may be numpy arrays
or torch tensors (CUDA tensors avoid the host->device copy).  For batched
device-resident work use ``kernels`` / ``verify_step`` directly.

These functions are API glue around the kernels and pay per-call host costs
the batched paths do not: numpy inputs are packed and copied to the device
per call, results come back to the host as dicts, ``verification_masks``
clamps on the host (``np.union1d`` per row), and ``sparse_attention`` ships
the whole K/V it is given to the device on every call.  They exist so a
reference caller can switch imports; the device pipelines
(``verify_step.STSVerifyStep``, ``specdec.generate``) keep everything resident.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import kernels
from .errors import ConfigError, ContractViolation
from .headmap import HeadKey, HeadMapping

SCOPE_DECODE = "decode"
SCOPE_PREFILL_DECODE = "prefill-decode"


@dataclass(frozen=True)
class SparsityConfig:
    """Budget, granularity and scope of mask generation (src/sparsity.py:33-69)."""

    budget: float
    page_size: int = 1
    scope: str = SCOPE_DECODE
    include_current: bool = True
    include_sink: bool = False
    recent_window: int = 0

    def __post_init__(self) -> None:
        if isinstance(self.budget, float) and not 0.0 < self.budget <= 1.0:
            raise ConfigError(f"fractional budget must be in (0, 1], got {self.budget}")
        if isinstance(self.budget, int) and self.budget < 1:
            raise ConfigError(f"token budget must be >= 1, got {self.budget}")
        if self.page_size < 1:
            raise ConfigError("page_size must be >= 1")
        if self.scope not in (SCOPE_DECODE, SCOPE_PREFILL_DECODE):
            raise ConfigError(f"unknown scope {self.scope!r}")
        if self.recent_window < 0:
            raise ConfigError("recent_window must be >= 0")

    def tokens_for_context(self, n: int) -> int:
        if isinstance(self.budget, int):
            return self.budget
        return max(1, math.ceil(self.budget * n))

    def sparse_prefill(self) -> bool:
        return self.scope == SCOPE_PREFILL_DECODE

    def select_kwargs(self) -> dict:
        return select_kwargs(self)


def select_kwargs(cfg) -> dict:
    """Selection arguments of any object with the reference ``SparsityConfig``
    fields (this class, or ``specsparse.sparsity.SparsityConfig`` itself,
    src/sparsity.py:33-59): the drop-in functions accept either."""
    return dict(budget=cfg.budget, page_size=cfg.page_size, include_current=cfg.include_current,
                include_sink=cfg.include_sink, recent_window=cfg.recent_window)


def _device():
    if not torch.cuda.is_available():
        raise RuntimeError("the STS B200 path needs a CUDA device (there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _pack_rows(rows, dev):
    """list of 1-D float rows -> (fp32 [R, maxlen] device tensor, int32 lengths),
    packed on the host (or on the device for CUDA rows) and copied once."""
    lens = [int(r.shape[0]) for r in rows]
    width = max(max(lens), 1)
    width = -(-width // 4) * 4
    if all(isinstance(r, torch.Tensor) and r.is_cuda for r in rows):
        buf = torch.zeros((len(rows), width), dtype=torch.float32, device=dev)
        for i, r in enumerate(rows):
            buf[i, : lens[i]] = r.to(dtype=torch.float32)
    else:
        host = np.zeros((len(rows), width), dtype=np.float32)
        for i, r in enumerate(rows):
            host[i, : lens[i]] = r.cpu().numpy() if isinstance(r, torch.Tensor) else np.asarray(r, dtype=np.float32)
        buf = torch.from_numpy(host).to(dev)
    return buf, torch.tensor(lens, dtype=torch.int32, device=dev)


def _unpack(idx, cnt):
    idx = idx.cpu().numpy()
    cnt = cnt.cpu().numpy()
    return [idx[i, : cnt[i]].astype(np.int64) for i in range(idx.shape[0])]


def select_rows(rows, cfg: SparsityConfig, tail_len: int = 0):
    """GPU _select_row over a list of rows (one launch); list of int64 arrays."""
    if not rows:
        return []
    dev = _device()
    buf, lens = _pack_rows(rows, dev)
    idx, cnt = kernels.select_topk(buf, row_len=lens, tail_len=tail_len, **select_kwargs(cfg))
    return _unpack(idx, cnt)


def page_aggregate(scores, page_size: int) -> np.ndarray:
    """fp64 page sums in numpy reduceat order (src/sparsity.py:72-83), on the GPU."""
    if page_size < 1:
        raise ContractViolation("page_size must be >= 1")
    from . import _lib

    arr = scores if isinstance(scores, torch.Tensor) else torch.from_numpy(np.asarray(scores, dtype=np.float32).ravel().copy())
    dev = _device()
    x = arr.to(device=dev, dtype=torch.float32).reshape(1, -1).contiguous()
    n = x.shape[1]
    pages = -(-n // page_size)
    out = torch.empty((1, max(pages, 1)), dtype=torch.float64, device=dev)
    if n > 0:
        _lib.call("sts_page_aggregate", x.data_ptr(), max(n, 1), 1, None, n, page_size, out.data_ptr(),
                  out.stride(0), _lib.stream_handle())
    return out[0, :pages].cpu().numpy()


def draft_masks_decode(rows: dict, cfg: SparsityConfig) -> dict:
    """One index set per draft head from its attention row (src/sparsity.py:115-119)."""
    heads = list(rows.keys())
    masks = select_rows([rows[h] for h in heads], cfg)
    return dict(zip(heads, masks))


def draft_masks_prefill(matrices: dict, cfg: SparsityConfig) -> dict:
    """Per-row masks over each causal prefix (src/sparsity.py:122-130); all
    rows of all heads in one launch."""
    flat, owners = [], []
    for head, mat in matrices.items():
        m = mat if isinstance(mat, torch.Tensor) else np.asarray(mat)
        for t in range(m.shape[0]):
            flat.append(m[t, : t + 1])
            owners.append(head)
    masks = select_rows(flat, cfg)
    out: dict = {h: [] for h in matrices}
    for h, m in zip(owners, masks):
        out[h].append(m)
    return out


def remap_masks(draft_masks: dict, mapping: HeadMapping) -> dict:
    """Copy each mapped draft head's mask to its target heads (src/sparsity.py:133-149).

    Host bookkeeping only (dict of copies); the device pipeline performs the
    same remap as an int32 indirection table (HeadMapping.to_table).
    """
    out: dict = {}
    for target, (draft, _) in mapping.entries.items():
        if draft not in draft_masks:
            raise ContractViolation(f"no draft mask for head {draft} (target {target})")
        value = draft_masks[draft]
        if isinstance(value, list):
            out[target] = [np.array(v, dtype=np.int64, copy=True) for v in value]
        else:
            out[target] = np.array(value, dtype=np.int64, copy=True)
    return out


def sparse_attention(q, keys, values, mask) -> np.ndarray:
    """Single-query attention over the masked subset (src/sparsity.py:152-173),
    computed by the fp32 gather kernel.  Slow path (API glue): copies the
    given K/V to the device on every call; batched callers use
    ``kernels.sparse_decode`` on resident caches."""
    idx = np.asarray(mask, dtype=np.int64).ravel()
    if idx.size == 0:
        raise ContractViolation("sparse attention needs a non-empty mask")
    n = keys.shape[0]
    if idx.min() < 0 or idx.max() >= n:
        raise ContractViolation("mask index outside the cached context")
    dev = _device()

    def dev32(x):
        t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.asarray(x, dtype=np.float32))
        return t.to(device=dev, dtype=torch.float32).contiguous()

    qd = dev32(q).reshape(1, 1, -1)
    kd = dev32(keys).reshape(1, n, -1)
    vd = dev32(values).reshape(1, n, -1)
    it = torch.from_numpy(idx.astype(np.int32)).to(dev).reshape(1, -1)
    cnt = torch.tensor([idx.size], dtype=torch.int32, device=dev)
    out, _ = kernels.sparse_decode(qd, kd, vd, idx=it, cnt=cnt, splits=1)
    return out[0, 0].cpu().numpy()


def sparse_prefill_attention(q, keys, values, row_masks, positions=None) -> np.ndarray:
    """Masked prefill attention of one head: row r (at position ``positions[r]``,
    default r) attends exactly ``row_masks[r]`` — the masked path of
    toymodel._run_block (src/toymodel.py:315-348, row validation
    ``_row_allowed`` :257-272) reached through forward_prefill(masks=...)
    with masks from draft_masks_prefill.  One fp32 kernel launch for all rows.
    Returns float32 [m, d]."""
    m = len(row_masks)
    n = keys.shape[0]
    pos = np.arange(m) if positions is None else np.asarray(positions, dtype=np.int64)
    lists = []
    for r, mr in enumerate(row_masks):
        idx = np.asarray(mr, dtype=np.int64).ravel()
        if idx.size == 0:
            raise ContractViolation(f"empty mask row at position {int(pos[r])}")
        if idx.min() < 0 or idx.max() > pos[r] or idx.max() >= n:
            raise ContractViolation(f"mask at position {int(pos[r])} escapes the causal prefix")
        lists.append(idx)
    dev = _device()
    width = max(len(x) for x in lists) if lists else 1
    idx_t = torch.zeros((m, width), dtype=torch.int32)
    cnt_t = torch.zeros((m,), dtype=torch.int32)
    for r, x in enumerate(lists):
        idx_t[r, : x.size] = torch.from_numpy(x.astype(np.int32))
        cnt_t[r] = x.size

    def dev32(x):
        t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.asarray(x, dtype=np.float32))
        return t.to(device=dev, dtype=torch.float32).contiguous()

    qd = dev32(q).reshape(1, m, 1, -1)
    kd = dev32(keys).reshape(1, n, -1)
    vd = dev32(values).reshape(1, n, -1)
    out, _ = kernels.sparse_prefill(qd, kd, vd, idx=idx_t.to(dev), cnt=cnt_t.to(dev))
    return out[0, :, 0].cpu().numpy()


def dump_masks(fh, step: int, masks: dict) -> None:
    """Append one JSON document describing a step's masks (src/sparsity.py:176-185)."""
    heads = {}
    for (layer, head), value in sorted(masks.items()):
        key = f"{layer}.{head}"
        if isinstance(value, list):
            heads[key] = [[int(i) for i in row] for row in value]
        else:
            heads[key] = [int(i) for i in value]
    fh.write(json.dumps({"step": step, "heads": heads}, sort_keys=True) + "\n")


def _clamp_current(indices, pos: int) -> np.ndarray:
    """src/specdec.py:212-216."""
    arr = np.asarray(indices, dtype=np.int64)
    arr = arr[arr <= pos]
    return np.union1d(arr, np.asarray([pos], dtype=np.int64))


def verification_masks(draft_rows: list, base: int, sparsity: SparsityConfig, mapping: HeadMapping) -> dict:
    """``specdec._verification_masks`` (src/specdec.py:219-233): every
    (speculative row, draft head) is selected in ONE kernel launch, then
    remapped to target heads and clamped to its row's position."""
    heads = list(draft_rows[0].keys())
    flat = [draft_rows[i][h] for i in range(len(draft_rows)) for h in heads]
    masks = select_rows(flat, sparsity)
    per_row = []
    for i in range(len(draft_rows)):
        dm = dict(zip(heads, masks[i * len(heads) : (i + 1) * len(heads)]))
        per_row.append({t: _clamp_current(m, base + i) for t, m in remap_masks(dm, mapping).items()})
    return {head: [per_row[i][head] for i in range(len(draft_rows))] for head in per_row[0]}
