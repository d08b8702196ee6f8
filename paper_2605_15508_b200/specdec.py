"""Integrated verify loop on the B200: greedy speculative
decoding with the draft-guided sparse mask lifecycle, device-resident.

Drop-in for ``specsparse.specdec`` (src/specdec.py): ``SpecConfig``,
``RoundOutcome``, ``GenerateStats``, ``GenerateResult``, ``ModelSession``,
``propose`` (:150-167), ``verify`` (:170-209), ``generate`` (:258-383) with
``event_log=`` / ``mask_dump=`` (:264-265, :334-335, :358-375) and
``greedy_generate`` (:386-400) — same arguments, results and exceptions.

Per round, everything stays on the device between one host sync:

* propose: gamma draft decodes; each greedy token is an on-device argmax fed
  straight into the next decode's embedding gather, and each decode records
  its attention rows (the draft-score capture) into device buffers;
* masks: all gamma rows x draft heads in ONE ``sts_select_topk`` launch (row
  lengths base+i+1, the reference tie rule); the head remap and the causal
  clamp are an int32 (target head, row) -> list table, no mask copies;
* verify: one masked target block (``sts_block_attention_f64``), the greedy
  check (argmax, first mismatch, correction token) on the device; the host
  reads back (proposal, accepted length, correction) — the one sync;
* rollback: cache lengths move (K/V beyond them are dead, overwritten later);
* correction: the draft's correction decode + its one-row selection, then
  the target's masked correction decode on a second CUDA stream, overlapped
  with the next round's proposal on the draft stream (``overlap=True``).

The numerics are the reference's (model.py: fp64 attention math, fp64
accumulating projections), so tokens, masks, statistics and the event log
match the reference's ``generate`` exactly (tests/test_gpu_specdec.py).
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np
import torch

from . import kernels
from .errors import CapacityError, ConfigError, ContractViolation, InputError
from .model import (DeviceMasks, ForwardRecord, PagedKVCache, _decode_to_row_masks, _device, ensure_paired,
                    host_masks_to_device, run_block_device, _records, _validate_tokens)
from .sparsity import dump_masks


@dataclass
class SpecConfig:
    """Speculation depth plus optional sparsity wiring (src/specdec.py:48-60)."""

    gamma: int = 4
    sparsity: object = None
    mappings: object = None

    def __post_init__(self) -> None:
        if self.gamma < 1:
            raise ConfigError("gamma must be >= 1")
        if self.sparsity is not None and self.mappings is None:
            raise ConfigError("sparsity requires a head mapping set")


@dataclass
class RoundOutcome:
    proposed: list
    accepted_len: int
    correction_token: int
    masks_used: int


@dataclass
class GenerateStats:
    rounds: int = 0
    proposed_total: int = 0
    accepted_total: int = 0
    masks_generated: int = 0
    masks_discarded: int = 0

    @property
    def acceptance_rate(self) -> float:
        return self.accepted_total / self.proposed_total if self.proposed_total else 0.0

    def to_dict(self) -> dict:
        return {"rounds": self.rounds, "proposed_total": self.proposed_total, "accepted_total": self.accepted_total,
                "acceptance_rate": self.acceptance_rate, "masks_generated": self.masks_generated,
                "masks_discarded": self.masks_discarded}


@dataclass
class GenerateResult:
    tokens: list
    new_tokens: list
    stats: GenerateStats
    rounds: list = field(default_factory=list)


def _tokens_for_context(cfg, n: int) -> int:
    """SparsityConfig.tokens_for_context (src/sparsity.py:62-66) on any
    object with the reference fields."""
    b = cfg.budget
    if isinstance(b, int):
        return b
    return max(1, math.ceil(b * n))


class ModelSession:
    """One model, its HBM-resident cache and the logits of the last processed
    position (src/specdec.py:100-137).  ``last_logits`` is a numpy view of the
    device row (the device row itself is ``last_logits_device``)."""

    def __init__(self, weights, device=None):
        self.weights = weights
        self.device = torch.device(device) if device is not None else _device()
        self.cache = PagedKVCache(weights.config, self.device)
        self.last_logits_device: torch.Tensor | None = None

    @property
    def last_logits(self):
        return None if self.last_logits_device is None else self.last_logits_device.cpu().numpy()

    @property
    def length(self) -> int:
        return self.cache.length

    def _run(self, tokens: torch.Tensor, masks=None, record_attention=False, status=None):
        logits, probs, _ = run_block_device(self.weights, tokens, self.cache, self.cache.length, masks=masks,
                                            record_attention=record_attention, status=status)
        self.last_logits_device = logits[-1]
        return logits, probs

    def prefill(self, tokens, *, masks=None, record_attention: bool = False) -> ForwardRecord:
        if self.cache.length != 0:
            raise ContractViolation("session already prefilled")
        cfg = self.weights.config
        arr = _validate_tokens(tokens, cfg.vocab)
        if arr.size < 1:
            raise InputError("prefill needs at least one token")
        if arr.size > cfg.max_seq:
            raise CapacityError(f"sequence of {arr.size} exceeds max_seq={cfg.max_seq}")
        return self._host_forward(arr, masks, record_attention)

    def decode(self, token: int, *, masks=None, record_attention: bool = False) -> ForwardRecord:
        arr = _validate_tokens([token], self.weights.config.vocab)
        return self._host_forward(arr, _decode_to_row_masks(masks, self.cache.length), record_attention)

    def block(self, tokens, *, masks=None) -> ForwardRecord:
        arr = _validate_tokens(tokens, self.weights.config.vocab)
        if arr.size < 1:
            raise InputError("block needs at least one token")
        return self._host_forward(arr, masks, False)

    def _host_forward(self, arr, masks, record_attention) -> ForwardRecord:
        cfg = self.weights.config
        start = self.cache.length
        m = int(arr.size)
        dm = host_masks_to_device(masks, cfg, m, start + np.arange(m), self.device) if masks else None
        logits, probs = self._run(torch.from_numpy(arr).to(self.device), dm, record_attention)
        return ForwardRecord(logits=logits.cpu().numpy(), start_pos=start, attention=_records(cfg, m, probs))

    def rollback(self, length: int) -> None:
        self.cache.truncate(length)


def propose(draft: ModelSession, gamma: int):
    """Draft ``gamma`` greedy tokens, recording each step's attention rows
    (src/specdec.py:150-167).  Returns (tokens, rows) like the reference."""
    toks, rows_dev = _propose_device(draft, gamma, record=True)
    cfg = draft.weights.config
    rows = []
    for i, r in enumerate(rows_dev):
        a = r.cpu().numpy()
        rows.append({(l, h): a[l * cfg.heads + h] for l in range(cfg.layers) for h in range(cfg.heads)})
    return [int(t) for t in toks.cpu().tolist()], rows


def _propose_device(draft: ModelSession, gamma: int, record: bool, status=None):
    """Device form of propose: (tokens int64 [gamma], rows: list of fp32
    [layers*heads, base+i+1] device tensors)."""
    if draft.last_logits_device is None:
        raise ContractViolation("draft session must be prefilled before proposing")
    if draft.length + gamma > draft.weights.config.max_seq:
        raise CapacityError("draft cache cannot hold the proposal")
    toks = torch.empty((gamma,), dtype=torch.int64, device=draft.device)
    rows = []
    for i in range(gamma):
        tok = torch.argmax(draft.last_logits_device).view(1)  # first max, like np.argmax
        toks[i : i + 1] = tok
        _, probs = draft._run(tok, record_attention=record, status=status)
        if record:
            rows.append(torch.cat(probs, 0))  # [layers*heads (x 1 row), n]
    return toks, rows


def verify(target: ModelSession, proposed, row_masks) -> RoundOutcome:
    """Check all proposed tokens in one (optionally sparse) forward
    (src/specdec.py:170-209)."""
    if target.last_logits_device is None:
        raise ContractViolation("target session must be prefilled before verifying")
    gamma = len(proposed)
    if row_masks is not None:
        cfg = target.weights.config
        for layer in range(cfg.layers):
            for head in range(cfg.heads):
                rows = row_masks.get((layer, head))
                if rows is None or len(rows) != gamma:
                    raise ContractViolation(f"verification masks do not cover head ({layer}, {head}) "
                                            f"for all {gamma} rows")
    base = target.length
    arr = _validate_tokens(proposed, target.weights.config.vocab)
    dm = host_masks_to_device(row_masks, target.weights.config, gamma, base + np.arange(gamma), target.device) \
        if row_masks else None
    acc, corr = _verify_device(target, torch.from_numpy(arr).to(target.device), dm)
    acc, corr = int(acc.item()), int(corr.item())
    target.rollback(base + acc)
    return RoundOutcome(proposed=[int(t) for t in proposed], accepted_len=acc, correction_token=corr,
                        masks_used=0 if row_masks is None else 1)


def _verify_device(target: ModelSession, proposed: torch.Tensor, masks, status=None):
    """The masked target block + greedy acceptance on the device; returns
    (accepted int64 [], correction int64 []) device scalars.  The caller rolls
    the cache back once the accepted length is on the host."""
    gamma = int(proposed.shape[0])
    boundary = target.last_logits_device
    logits, _ = target._run(proposed, masks, status=status)
    greedy = torch.argmax(torch.cat([boundary.view(1, -1), logits], 0), dim=1)  # [gamma + 1]
    match = (proposed == greedy[:gamma]).to(torch.int64)
    acc = torch.cumprod(match, 0).sum()
    return acc, greedy[acc]


def _clamp_current(indices, pos: int) -> np.ndarray:
    arr = np.asarray(indices, dtype=np.int64)
    arr = arr[arr <= pos]
    return np.union1d(arr, np.asarray([pos], dtype=np.int64))


def _touched_pages(length: int, config, masks_per_row):
    """Per layer, sorted [head, page] pairs the round's target pass touched
    (src/specdec.py:236-255, the offload simulator's wire format)."""
    p_s = config.page_size
    touched = [set() for _ in range(config.layers)]
    if masks_per_row is None:
        pages = range(-(-length // p_s))
        for layer in range(config.layers):
            touched[layer] = {(h, p) for h in range(config.heads) for p in pages}
    else:
        for masks in masks_per_row:
            for (layer, head), value in masks.items():
                rows = value if isinstance(value, list) else [value]
                for idx in rows:
                    for p in set(int(i) // p_s for i in np.asarray(idx).ravel()):
                        touched[layer].add((head, p))
    return [[list(pair) for pair in sorted(t)] for t in touched]


class _MaskBuilder:
    """Device mask build of one round: the gamma proposal rows (or the
    correction row) x every draft head in one select launch, plus the int32
    (target layer, head, row) -> list table of the round's mapping."""

    def __init__(self, sparsity, draft_cfg, target_cfg, device):
        self.s = sparsity
        self.dcfg, self.tcfg = draft_cfg, target_cfg
        self.dev = device
        self.Nd = draft_cfg.layers * draft_cfg.heads
        self._tables = {}

    def table(self, mapping, m: int, prefill: bool = False) -> torch.Tensor:
        """lor[l, h*m + r] = list of (target (l, h), row r): decode/verify rows
        are stacked row-major over draft heads (r*Nd + j), prefill rows
        head-major (j*m + r)."""
        key = (id(mapping), m, prefill)
        t = self._tables.get(key)
        if t is None:
            L, H = self.tcfg.layers, self.tcfg.heads
            lor = np.empty((L, H * m), dtype=np.int32)
            for l in range(L):
                for h in range(H):
                    try:
                        dl, dh = mapping.entries[(l, h)][0]
                    except KeyError:
                        raise ContractViolation(f"mapping has no entry for target head {(l, h)}") from None
                    j = dl * self.dcfg.heads + dh
                    for r in range(m):
                        lor[l, h * m + r] = j * m + r if prefill else r * self.Nd + j
            t = self._tables[key] = torch.from_numpy(lor).to(self.dev)
        return t

    def select(self, rows, lens, status=None):
        """rows: list of fp32 device [Nd, n_i] blocks (row lengths lens[i]);
        returns (idx, cnt) over the stacked rows (block i, head j) = i*Nd + j."""
        width = -(-max(lens) // 4) * 4
        buf = torch.zeros((len(rows) * self.Nd, width), dtype=torch.float32, device=self.dev)
        row_len = torch.empty((len(rows) * self.Nd,), dtype=torch.int32, device=self.dev)
        for i, (r, n) in enumerate(zip(rows, lens)):
            buf[i * self.Nd : (i + 1) * self.Nd, :n] = r[:, :n]
            row_len[i * self.Nd : (i + 1) * self.Nd] = n
        s = self.s
        return kernels.select_topk(buf, row_len=row_len, budget=s.budget, page_size=s.page_size,
                                   include_current=s.include_current, include_sink=s.include_sink,
                                   recent_window=s.recent_window, status=status)


def _host_lists(idx: torch.Tensor, cnt: torch.Tensor):
    ih, ch = idx.cpu().numpy(), cnt.cpu().numpy()
    return [ih[i, : ch[i]].astype(np.int64) for i in range(ih.shape[0])]


def generate(draft_weights, target_weights, prompt, max_new: int, cfg, event_log=None, mask_dump=None,
             overlap: bool = True) -> GenerateResult:
    """Speculative generation loop: propose, mask, verify, commit
    (src/specdec.py:258-296).  ``overlap``: run the target's correction decode
    on a second stream, concurrent with the next round's proposal."""
    prompt = [int(t) for t in prompt]
    if not prompt:
        raise InputError("prompt must not be empty")
    if max_new < 1:
        raise InputError("max_new must be >= 1")
    ensure_paired(draft_weights.config, target_weights.config)
    limit = min(draft_weights.config.max_seq, target_weights.config.max_seq)
    if len(prompt) + max_new + cfg.gamma + 1 > limit:
        raise CapacityError(f"prompt {len(prompt)} + max_new {max_new} + gamma {cfg.gamma} + 1 "
                            f"exceeds max_seq {limit}")
    own_log = isinstance(event_log, (str, Path))
    log_fh = open(event_log, "w") if own_log else event_log
    try:
        return _generate_inner(draft_weights, target_weights, prompt, max_new, cfg, log_fh, mask_dump, overlap)
    finally:
        if own_log and log_fh is not None:
            log_fh.close()


def _generate_inner(draft_weights, target_weights, prompt, max_new, cfg, log_fh, mask_dump, overlap):
    dev = _device()
    draft = ModelSession(draft_weights, dev)
    target = ModelSession(target_weights, dev)
    dcfg, tcfg = draft_weights.config, target_weights.config
    sparsity = cfg.sparsity
    gamma = cfg.gamma
    status = torch.zeros((1,), dtype=torch.int32, device=dev)
    mb = _MaskBuilder(sparsity, dcfg, tcfg, dev) if sparsity is not None else None
    s_draft = torch.cuda.current_stream(dev)
    s_target = torch.cuda.Stream(device=dev) if overlap else s_draft

    p = torch.tensor(prompt, dtype=torch.int64, device=dev)
    if sparsity is not None and sparsity.scope == "prefill-decode":
        _, probs = draft._run(p, record_attention=True, status=status)
        n = len(prompt)
        mapping = cfg.mappings.nearest(_tokens_for_context(sparsity, n))
        rows = torch.cat(probs, 0)  # [Nd * n, n]: (draft head j, row t)
        row_len = torch.arange(1, n + 1, dtype=torch.int32, device=dev).repeat(mb.Nd)
        width = -(-n // 4) * 4
        buf = torch.zeros((rows.shape[0], width), dtype=torch.float32, device=dev)
        buf[:, :n] = rows
        s = sparsity
        idx, cnt = kernels.select_topk(buf, row_len=row_len, budget=s.budget, page_size=s.page_size,
                                       include_current=s.include_current, include_sink=s.include_sink,
                                       recent_window=s.recent_window, status=status)
        target._run(p, DeviceMasks(idx, cnt, mb.table(mapping, n, prefill=True)), status=status)
    else:
        draft._run(p, status=status)
        target._run(p, status=status)

    committed = list(prompt)
    stats = GenerateStats()
    outcomes = []
    want_masks = log_fh is not None or mask_dump is not None
    while len(committed) - len(prompt) < max_new:
        base = target.length
        # proposal (draft stream): device argmax chain + recorded rows
        proposed, rows = _propose_device(draft, gamma, record=sparsity is not None, status=status)
        row_masks_dev = None
        mapping = None
        if sparsity is not None:
            mapping = cfg.mappings.nearest(_tokens_for_context(sparsity, base + 1))
            # exact draft masks (the configured extras); every row also attends its
            # own position (specdec._clamp_current) inside the attention kernel
            idx, cnt = mb.select(rows, [base + i + 1 for i in range(gamma)], status=status)
            row_masks_dev = DeviceMasks(idx, cnt, mb.table(mapping, gamma), include_self=True)
            stats.masks_generated += 1
        # verify (target stream, after the proposal and the previous correction decode)
        s_target.wait_stream(s_draft)
        with torch.cuda.stream(s_target):
            acc_t, corr_t = _verify_device(target, proposed, row_masks_dev, status=status)
            res = torch.cat([proposed, acc_t.view(1), corr_t.view(1)]).cpu()  # the round's one sync
        s_draft.wait_stream(s_target)
        res = res.tolist()
        prop_h, acc, corr = [int(t) for t in res[:gamma]], int(res[gamma]), int(res[gamma + 1])
        target.rollback(base + acc)
        outcome = RoundOutcome(proposed=prop_h, accepted_len=acc, correction_token=corr,
                               masks_used=0 if sparsity is None else 1)
        stats.rounds += 1
        stats.proposed_total += gamma
        stats.accepted_total += acc
        if sparsity is not None and acc < gamma:
            stats.masks_discarded += 1

        row_masks = None
        if want_masks and sparsity is not None:
            lists = _host_lists(row_masks_dev.idx, row_masks_dev.cnt)
            row_masks = {}
            for (tl, th), (dh_key, _) in sorted(mapping.entries.items()):
                j = dh_key[0] * dcfg.heads + dh_key[1]
                row_masks[(tl, th)] = [_clamp_current(lists[i * mb.Nd + j], base + i) for i in range(gamma)]
            if mask_dump is not None:
                dump_masks(mask_dump, stats.rounds - 1, row_masks)

        # correction: draft decode (+ its one-row selection) on the draft stream,
        # then the target's masked decode on the target stream
        draft.rollback(len(committed) + acc)
        ctok = torch.tensor([corr], dtype=torch.int64, device=dev)
        _, cprobs = draft._run(ctok, record_attention=sparsity is not None, status=status)
        corr_dev = None
        corr_masks = None
        if sparsity is not None:
            n = draft.length
            cidx, ccnt = mb.select([torch.cat(cprobs, 0)], [n], status=status)
            corr_dev = DeviceMasks(cidx, ccnt, mb.table(mapping, 1), include_self=True)  # decode: mask ∪ {current}
            if want_masks:
                cl = _host_lists(cidx, ccnt)
                corr_masks = {t: cl[d[0] * dcfg.heads + d[1]] for t, (d, _) in mapping.entries.items()}
        s_target.wait_stream(s_draft)
        with torch.cuda.stream(s_target):
            target._run(ctok, corr_dev, status=status)
            if corr_dev is not None:
                for t in (corr_dev.idx, corr_dev.cnt):
                    t.record_stream(s_target)
        committed.extend(prop_h[:acc])
        committed.append(corr)
        outcomes.append(outcome)

        if log_fh is not None:
            mask_trace = [row_masks, corr_masks] if row_masks is not None else None
            record = {
                "round": stats.rounds - 1, "context_len": base, "proposed": prop_h, "accepted_len": acc,
                "correction": corr,
                "budget": _tokens_for_context(sparsity, base + 1) if sparsity is not None else None,
                "pages_touched": _touched_pages(target.length, tcfg, mask_trace),
            }
            log_fh.write(json.dumps(record, sort_keys=True) + "\n")
    torch.cuda.current_stream(dev).wait_stream(s_target)
    st = int(status.item())
    if st:
        raise ContractViolation(f"device status {st:#x} during generation (bad or empty mask row)")
    new_tokens = committed[len(prompt):][:max_new]
    return GenerateResult(tokens=prompt + new_tokens, new_tokens=new_tokens, stats=stats, rounds=outcomes)


def greedy_generate(weights, prompt, max_new: int) -> list:
    """Plain target-only greedy decoding, the losslessness reference
    (src/specdec.py:386-400); the argmax chain stays on the device."""
    prompt = [int(t) for t in prompt]
    if not prompt:
        raise InputError("prompt must not be empty")
    if len(prompt) + max_new > weights.config.max_seq:
        raise CapacityError("sequence would exceed max_seq")
    session = ModelSession(weights)
    status = torch.zeros((1,), dtype=torch.int32, device=session.device)
    session._run(torch.tensor(prompt, dtype=torch.int64, device=session.device), status=status)
    out = torch.empty((max_new,), dtype=torch.int64, device=session.device)
    for i in range(max_new):
        tok = torch.argmax(session.last_logits_device).view(1)
        out[i : i + 1] = tok
        session._run(tok, status=status)
    return prompt + [int(t) for t in out.cpu().tolist()]
