"""Reference-named model-level entry points on the B200: the capture and
verify forwards the STS path is reached through.

Drop-in for ``specsparse.toymodel``'s forward surface (src/toymodel.py):
``ModelConfig`` (:38-77), ``ForwardRecord`` (:226-240), ``PagedKVCache``
(:163-222, device-resident here), ``forward_prefill`` / ``forward_decode`` /
``forward_block`` (:359-455) with ``masks=``, ``record_attention=`` and
``record_scores=``.  Same arguments, return types (numpy logits, dicts of
fp32 numpy attention / score matrices keyed (layer, head)) and exceptions.

What runs where:

* the attention of every head of a layer — causal or masked per row, the
  recorded softmax rows (``ForwardRecord.attention``, the draft-score capture
  of ``specdec.propose``, src/specdec.py:150-167) and the raw scores
  (``ForwardRecord.scores``) — is ONE launch of ``sts_block_attention_f64``
  (include/sts_b200.h), fp64 math as the reference states it, so recorded
  rows, the masks selected from them and the greedy tokens are the
  reference's own;
* K/V live in HBM (``PagedKVCache`` here keeps [layers][heads][max_seq][d]
  fp32 device tensors; a reference ``PagedKVCache`` passed in is written
  through and mirrored);
* the non-attention plumbing of the toy model (embeddings, RMS norms,
  projections, ReLU MLP, LM head — SURVEY §2 marks the toy model out of
  scope) runs as torch fp64 ops on the same device, mirroring the reference's
  float discipline (fp64 accumulation, fp32 storage; src/numkit.py:29-40,
  src/toymodel.py:243-246).

There is no CPU path: without a CUDA device every entry point raises.
"""

from __future__ import annotations

import math
import weakref
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr, stream_handle
from .errors import CapacityError, ConfigError, ContractViolation, InputError

HeadKey = tuple[int, int]
_NORM_EPS = 1e-6


@dataclass(frozen=True)
class ModelConfig:
    """Shape and seed of a toy model (src/toymodel.py:38-77)."""

    layers: int
    heads: int
    head_dim: int
    vocab: int
    max_seq: int
    page_size: int = 4
    mlp_ratio: int = 4
    seed: int = 0

    def __post_init__(self) -> None:
        for name in ("layers", "heads", "head_dim", "vocab", "max_seq", "page_size", "mlp_ratio"):
            if getattr(self, name) < 1:
                raise ConfigError(f"ModelConfig.{name} must be >= 1")

    @property
    def hidden(self) -> int:
        return self.heads * self.head_dim

    def to_dict(self) -> dict:
        return {k: getattr(self, k) for k in ("layers", "heads", "head_dim", "vocab", "max_seq", "page_size",
                                               "mlp_ratio", "seed")}

    @classmethod
    def from_dict(cls, d: dict) -> "ModelConfig":
        try:
            return cls(**{k: int(d[k]) for k in cls.__dataclass_fields__ if k in d})
        except (KeyError, TypeError, ValueError) as exc:
            raise InputError(f"bad model config: {exc}") from exc


def ensure_paired(draft, target) -> None:
    """src/toymodel.py:80-86."""
    if draft.vocab != target.vocab or draft.max_seq != target.max_seq:
        raise InputError(
            "draft and target models must share vocab and max_seq: "
            f"({draft.vocab}, {draft.max_seq}) vs ({target.vocab}, {target.max_seq})")


@dataclass
class ForwardRecord:
    """Logits plus optional attention / score recordings (src/toymodel.py:226-240)."""

    logits: np.ndarray
    start_pos: int
    attention: dict | None = None
    scores: dict | None = None


def _device():
    if not torch.cuda.is_available():
        raise RuntimeError("the STS B200 path needs a CUDA device (there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


class PagedKVCache:
    """Device-resident per-layer K/V with the reference cache interface
    (src/toymodel.py:163-222): length, pages, residency tier tags (which never
    affect results), write/advance/truncate.  Storage is head-major fp32
    [layers][heads][max_seq][head_dim] in HBM, one tensor each for K and V."""

    def __init__(self, config, device=None):
        self.config = config
        dev = torch.device(device) if device is not None else _device()
        shape = (config.layers, config.heads, config.max_seq, config.head_dim)
        self.k = torch.zeros(shape, dtype=torch.float32, device=dev)
        self.v = torch.zeros(shape, dtype=torch.float32, device=dev)
        self.length = 0
        self._slow_pages: set = set()

    @property
    def page_size(self) -> int:
        return self.config.page_size

    @property
    def page_count(self) -> int:
        return -(-self.length // self.config.page_size)

    def keys(self, layer: int, upto: int | None = None) -> np.ndarray:
        n = self.length if upto is None else upto
        return self.k[layer, :, :n].permute(1, 0, 2).cpu().numpy()

    def values(self, layer: int, upto: int | None = None) -> np.ndarray:
        n = self.length if upto is None else upto
        return self.v[layer, :, :n].permute(1, 0, 2).cpu().numpy()

    def write_block(self, layer: int, start: int, k, v) -> None:
        kt = torch.as_tensor(k, dtype=torch.float32).to(self.k.device)
        vt = torch.as_tensor(v, dtype=torch.float32).to(self.k.device)
        m = kt.shape[0]
        self.k[layer, :, start : start + m] = kt.permute(1, 0, 2)
        self.v[layer, :, start : start + m] = vt.permute(1, 0, 2)

    def advance(self, m: int) -> None:
        if self.length + m > self.config.max_seq:
            raise CapacityError(f"cache full: {self.length}+{m} exceeds max_seq={self.config.max_seq}")
        self.length += m

    def truncate(self, n: int) -> None:
        if not 0 <= n <= self.length:
            raise ContractViolation(f"cannot truncate cache of length {self.length} to {n}")
        self.length = n
        self._slow_pages = {t for t in self._slow_pages if t[2] < self.page_count}

    def tier(self, layer: int, head: int, page: int) -> str:
        self._check_page(layer, head, page)
        return "slow" if (layer, head, page) in self._slow_pages else "fast"

    def set_tier(self, layer: int, head: int, page: int, tier: str) -> None:
        self._check_page(layer, head, page)
        if tier not in ("fast", "slow"):
            raise ContractViolation(f"unknown tier {tier!r}")
        if tier == "slow":
            self._slow_pages.add((layer, head, page))
        else:
            self._slow_pages.discard((layer, head, page))

    def _check_page(self, layer: int, head: int, page: int) -> None:
        cfg = self.config
        if not (0 <= layer < cfg.layers and 0 <= head < cfg.heads and 0 <= page < self.page_count):
            raise ContractViolation(f"no page ({layer}, {head}, {page}) in cache")


# -- weights on the device (fp32 storage, fp64 copies of the matrices) -------------
_WEIGHTS: dict = {}
_MATS = ("wq", "wk", "wv", "wo", "w_up", "w_down", "lm_head")
_VECS = ("token_emb", "pos_emb", "attn_norm", "mlp_norm", "final_norm")


def device_weights(weights, device=None) -> dict:
    """The model's parameters as device tensors (cached per weights object):
    fp64 matrices for the fp64-accumulating projections, fp32 embeddings and
    norm scales as the reference stores them."""
    key = id(weights)
    hit = _WEIGHTS.get(key)
    if hit is not None and hit[0]() is weights:
        return hit[1]
    dev = torch.device(device) if device is not None else _device()
    d = {}
    for name in _MATS:
        d[name] = torch.from_numpy(np.asarray(getattr(weights, name), dtype=np.float64)).to(dev)
    for name in _VECS:
        d[name] = torch.from_numpy(np.asarray(getattr(weights, name), dtype=np.float32)).to(dev)
    try:
        ref = weakref.ref(weights, lambda _r, k=key: _WEIGHTS.pop(k, None))
    except TypeError:  # not weak-referenceable: keep it alive with the cache entry
        ref = (lambda w=weights: w)
    _WEIGHTS[key] = (ref, d)
    return d


def _mm(a: torch.Tensor, b64: torch.Tensor) -> torch.Tensor:
    """numkit.matmul (src/numkit.py:29-40): fp64 accumulation, fp32 result."""
    out = (a.double() @ b64).float()
    if not torch.isfinite(out).all():
        raise ContractViolation("matmul overflowed to non-finite values")
    return out


def _rms_norm(x: torch.Tensor, scale: torch.Tensor) -> torch.Tensor:
    """src/toymodel.py:243-246."""
    x64 = x.double()
    rms = torch.sqrt(torch.mean(x64 * x64, dim=-1, keepdim=True) + _NORM_EPS)
    return ((x64 / rms) * scale.double()).float()


def _validate_tokens(tokens, vocab: int) -> np.ndarray:
    arr = np.asarray(tokens, dtype=np.int64).ravel()
    if arr.size and (arr.min() < 0 or arr.max() >= vocab):
        bad = int(arr[(arr < 0) | (arr >= vocab)][0])
        raise InputError(f"token id {bad} outside vocabulary of size {vocab}")
    return arr


class DeviceMasks:
    """Per-(head, row) key lists for one block, already on the device: for
    layer l, row (h, r) uses list ``list_of_row[l][h*m + r]`` of ``idx``/``cnt``
    (-1: dense causal).  The device generate loop builds these straight from
    the select kernel's output (no host round trip)."""

    def __init__(self, idx: torch.Tensor, cnt: torch.Tensor, list_of_row: torch.Tensor, include_self: bool = False):
        self.idx, self.cnt, self.list_of_row = idx, cnt, list_of_row  # list_of_row [layers, heads*m]
        self.include_self = include_self  # listed rows also attend their own position


def host_masks_to_device(masks: dict, cfg, m: int, positions, dev) -> DeviceMasks:
    """Validate a reference masks dict (src/toymodel.py:257-272, :304-311) and
    lay it out as device key lists."""
    lists, lor = [], np.full((cfg.layers, cfg.heads * m), -1, dtype=np.int32)
    for (layer, head), rows in masks.items():
        if not (0 <= layer < cfg.layers and 0 <= head < cfg.heads):
            raise ContractViolation(f"mask refers to unknown head ({layer}, {head})")
        if len(rows) != m:
            raise ContractViolation(f"mask for head ({layer}, {head}) covers {len(rows)} rows, block has {m}")
        for r in range(m):
            pos = int(positions[r])
            idx = np.asarray(rows[r], dtype=np.int64).ravel()
            if idx.size == 0:
                raise ContractViolation(f"empty mask row for head ({layer}, {head}) at position {pos}")
            if idx.min() < 0 or idx.max() > pos:
                raise ContractViolation(f"mask for head ({layer}, {head}) at position {pos} escapes the causal prefix")
            lor[layer, head * m + r] = len(lists)
            lists.append(np.unique(idx))
    width = max((x.size for x in lists), default=1)
    idx_h = np.zeros((max(len(lists), 1), width), dtype=np.int32)
    cnt_h = np.zeros((max(len(lists), 1),), dtype=np.int32)
    for i, x in enumerate(lists):
        idx_h[i, : x.size] = x
        cnt_h[i] = x.size
    return DeviceMasks(torch.from_numpy(idx_h).to(dev), torch.from_numpy(cnt_h).to(dev), torch.from_numpy(lor).to(dev))


def block_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, start_pos: int, *, masks=None,
                    record_attention=False, record_scores=False, status=None, stream=None):
    """One layer's attention for every head: q fp32 [H, m, d], k/v fp32
    [H, >= start_pos + m, d] views (unit inner stride).  ``masks``: None or
    (idx, cnt, list_of_row [H*m]).  Returns (out fp32 [m, H*d], probs
    [H*m, n_end] or None, scores or None) — sts_block_attention_f64."""
    H, m, d = q.shape
    n_end = start_pos + m
    dev = q.device
    out = torch.empty((m, H * d), dtype=torch.float32, device=dev)
    probs = torch.empty((H * m, n_end), dtype=torch.float32, device=dev) if record_attention else None
    scores = torch.empty((H * m, n_end), dtype=torch.float32, device=dev) if record_scores else None
    rec_ld = n_end
    idx = cnt = lor = None
    flags = 0
    if masks is not None:
        idx, cnt, lor = masks[:3]
        flags = _lib.STS_BLOCK_INCLUDE_SELF if len(masks) > 3 and masks[3] else 0
    if k.stride(-1) != 1 or v.stride() != k.stride():
        raise ValueError("k/v must be [H, N, d] views with unit inner stride and equal strides")
    call("sts_block_attention_f64", ptr(q.contiguous()), ptr(k), ptr(v), k.stride(0), k.stride(1), H, m, d,
         start_pos, 1.0 / math.sqrt(d), ptr(idx), idx.stride(0) if idx is not None else 0, ptr(cnt), ptr(lor), flags,
         ptr(out), out.stride(0), ptr(probs), ptr(scores), rec_ld, ptr(status), stream_handle(stream))
    return out, probs, scores


def _kv_views(cache, layer: int, n_end: int, dev):
    """Device [H, n_end, d] K/V views of ``layer`` (a reference numpy cache is
    uploaded: its host arrays are the state)."""
    if isinstance(cache, PagedKVCache):
        return cache.k[layer, :, :n_end], cache.v[layer, :, :n_end]
    kh = np.ascontiguousarray(np.asarray(cache.keys(layer, n_end)).transpose(1, 0, 2), dtype=np.float32)
    vh = np.ascontiguousarray(np.asarray(cache.values(layer, n_end)).transpose(1, 0, 2), dtype=np.float32)
    return torch.from_numpy(kh).to(dev), torch.from_numpy(vh).to(dev)


def run_block_device(weights, tokens: torch.Tensor, cache, start_pos: int, *, masks: DeviceMasks | None = None,
                     record_attention=False, record_scores=False, append=True, status=None, stream=None):
    """The device form of ``_run_block`` (src/toymodel.py:275-356): ``tokens``
    int64 device tensor [m]; returns (logits fp32 [m, vocab], probs per layer
    [H*m, n_end] or None, scores per layer or None), all on the device.
    ``status``: a device int32 word the kernels OR their error bits into (the
    caller checks it); None = a private word checked here (one sync)."""
    cfg = weights.config
    m = int(tokens.shape[0])
    n_end = start_pos + m
    if append and start_pos != cache.length:
        raise ContractViolation("append block must start at the cache tail")
    if append and n_end > cfg.max_seq:
        raise CapacityError(f"cache full: {start_pos}+{m} exceeds max_seq={cfg.max_seq}")
    if not append and cache.length < n_end:
        raise ContractViolation("replay block extends past cached positions")
    W = device_weights(weights, tokens.device)
    dev = tokens.device
    H, d = cfg.heads, cfg.head_dim
    x = W["token_emb"][tokens] + W["pos_emb"][start_pos:n_end]
    probs_l, scores_l = [], []
    own_status = status is None
    if own_status:
        status = torch.zeros((1,), dtype=torch.int32, device=dev)
    for layer in range(cfg.layers):
        h = _rms_norm(x, W["attn_norm"][layer])
        q = _mm(h, W["wq"][layer]).reshape(m, H, d)
        k_new = _mm(h, W["wk"][layer]).reshape(m, H, d)
        v_new = _mm(h, W["wv"][layer]).reshape(m, H, d)
        if append:
            if isinstance(cache, PagedKVCache):
                cache.k[layer, :, start_pos:n_end] = k_new.permute(1, 0, 2)
                cache.v[layer, :, start_pos:n_end] = v_new.permute(1, 0, 2)
            else:  # reference cache: write through (its numpy arrays are the state)
                cache.write_block(layer, start_pos, k_new.cpu().numpy(), v_new.cpu().numpy())
        kv, vv = _kv_views(cache, layer, n_end, dev)
        mk = None
        if masks is not None:
            mk = (masks.idx, masks.cnt, masks.list_of_row[layer], masks.include_self)
        attn_out, probs, scores = block_attention(q.permute(1, 0, 2).contiguous(), kv, vv, start_pos, masks=mk,
                                                  record_attention=record_attention, record_scores=record_scores,
                                                  status=status, stream=stream)
        probs_l.append(probs)
        scores_l.append(scores)
        x = x + _mm(attn_out, W["wo"][layer])
        h2 = _rms_norm(x, W["mlp_norm"][layer])
        up = torch.clamp_min(_mm(h2, W["w_up"][layer]), 0.0)
        x = x + _mm(up, W["w_down"][layer])
    if append:
        cache.advance(m)
    logits = _mm(_rms_norm(x, W["final_norm"]), W["lm_head"])
    st = int(status.item()) if own_status else 0
    if st:
        raise ContractViolation(f"device status {st:#x} in block attention (bad or empty mask row)")
    return logits, (probs_l if record_attention else None), (scores_l if record_scores else None)


def _records(cfg, m: int, per_layer):
    if per_layer is None:
        return None
    out = {}
    for layer, t in enumerate(per_layer):
        a = t.cpu().numpy().reshape(cfg.heads, m, -1)
        for head in range(cfg.heads):
            out[(layer, head)] = a[head]
    return out


def _forward(weights, arr: np.ndarray, cache, start_pos: int, masks, record_attention, record_scores,
             append=True) -> ForwardRecord:
    cfg = weights.config
    dev = cache.k.device if isinstance(cache, PagedKVCache) else _device()
    m = int(arr.size)
    dm = None
    if masks:
        dm = host_masks_to_device(masks, cfg, m, start_pos + np.arange(m), dev)
    tokens = torch.from_numpy(arr).to(dev)
    logits, probs, scores = run_block_device(weights, tokens, cache, start_pos, masks=dm,
                                             record_attention=record_attention, record_scores=record_scores,
                                             append=append)
    return ForwardRecord(logits=logits.cpu().numpy(), start_pos=start_pos, attention=_records(cfg, m, probs),
                         scores=_records(cfg, m, scores))


def forward_prefill(weights, tokens, *, masks=None, record_attention: bool = False, record_scores: bool = False):
    """Causal forward over a fresh sequence (src/toymodel.py:359-384); returns
    (ForwardRecord, PagedKVCache) with the cache resident in HBM."""
    cfg = weights.config
    arr = _validate_tokens(tokens, cfg.vocab)
    if arr.size < 1:
        raise InputError("prefill needs at least one token")
    if arr.size > cfg.max_seq:
        raise CapacityError(f"sequence of {arr.size} exceeds max_seq={cfg.max_seq}")
    cache = PagedKVCache(cfg)
    rec = _forward(weights, arr, cache, 0, masks, record_attention, record_scores)
    return rec, cache


def _decode_to_row_masks(masks, pos: int):
    """src/toymodel.py:467-475: decode masks always include the current position."""
    if masks is None:
        return None
    return {key: [np.union1d(np.asarray(idx, dtype=np.int64), np.asarray([pos], dtype=np.int64))]
            for key, idx in masks.items()}


def forward_decode(weights, token: int, cache, *, masks=None, record_attention: bool = False,
                   record_scores: bool = False) -> ForwardRecord:
    """Append one token and return its logits row (src/toymodel.py:387-405)."""
    arr = _validate_tokens([token], weights.config.vocab)
    pos = cache.length
    return _forward(weights, arr, cache, pos, _decode_to_row_masks(masks, pos), record_attention, record_scores)


def forward_block(weights, tokens, cache, *, masks=None, record_attention: bool = False,
                  record_scores: bool = False) -> ForwardRecord:
    """Multi-token causal forward appended to the cache (src/toymodel.py:408-431)."""
    arr = _validate_tokens(tokens, weights.config.vocab)
    if arr.size < 1:
        raise InputError("block needs at least one token")
    return _forward(weights, arr, cache, cache.length, masks, record_attention, record_scores)


def replay_position(weights, cache, position: int, token: int, *, masks=None) -> np.ndarray:
    """Recompute the logits of one cached position, read-only (src/toymodel.py:434-455)."""
    if not 0 <= position < cache.length:
        raise ContractViolation(f"position {position} not in cache of length {cache.length}")
    arr = _validate_tokens([token], weights.config.vocab)
    rec = _forward(weights, arr, cache, position, _decode_to_row_masks(masks, position), False, False,
                   append=False)
    return rec.logits[0]


__all__ = [
    "ForwardRecord", "ModelConfig", "PagedKVCache", "block_attention", "device_weights", "ensure_paired",
    "forward_block", "forward_decode", "forward_prefill", "replay_position", "run_block_device",
]
_ = _lib  # the library is loaded by the first call through ``call``
