"""GPU parity of mask construction: sts_select_topk / sts_page_aggregate vs
the oracle and the reference golden vectors — bit-exact index sets."""

import json
import math

import numpy as np
import pytest

from conftest import cfg_from_json, load_golden, unpack
from oracle import sts_oracle as O

pytestmark = pytest.mark.gpu


def _rows_kind(rng, n, kind):
    if kind == "softmax":
        z = 2.0 * rng.standard_normal(n)
        w = np.exp(z - z.max())
        return (w / w.sum()).astype(np.float32)
    if kind == "ties":
        z = 2.0 * rng.standard_normal(n)
        w = np.exp(z - z.max())
        return (np.round((w / w.sum()) * 256) / 256).astype(np.float32)
    if kind == "coarse":
        return (rng.integers(0, 4, n) / 4.0).astype(np.float32)
    if kind == "special":
        x = rng.standard_normal(n).astype(np.float32)
        m = rng.random(n)
        x[m < 0.05] = np.nan
        x[(m >= 0.05) & (m < 0.1)] = -0.0
        x[(m >= 0.1) & (m < 0.15)] = 0.0
        x[(m >= 0.15) & (m < 0.17)] = np.inf
        x[(m >= 0.17) & (m < 0.19)] = -np.inf
        return x
    raise ValueError(kind)


def test_golden_topk_through_select(cuda_ok):
    from paper_2605_15508_b200 import SparsityConfig
    from paper_2605_15508_b200.sparsity import select_rows

    g = load_golden("topk.npz")
    rows = unpack(g["rows"], g["row_offs"])
    outs = unpack(g["out"], g["out_offs"])
    # topk_indices(row, k) == _select_row with int budget k, no extras, when k < n
    by_k = {}
    for r, k, want in zip(rows, g["k"], outs):
        by_k.setdefault(int(k), []).append((r, want))
    for k, items in by_k.items():
        cfg = SparsityConfig(budget=int(k), include_current=False)
        got = select_rows([r for r, _ in items], cfg)
        for (r, want), mask in zip(items, got):
            np.testing.assert_array_equal(mask, want)


def test_golden_select_row(cuda_ok):
    from paper_2605_15508_b200 import SparsityConfig, draft_masks_decode

    g = load_golden("select_row.npz")
    rows = unpack(g["rows"], g["row_offs"])
    outs = unpack(g["out"], g["out_offs"])
    for r, c, want in zip(rows, json.loads(str(g["cfg"])), outs):
        budget, ps, cur, sink, win = cfg_from_json(c)
        cfg = SparsityConfig(budget=budget, page_size=ps, include_current=cur, include_sink=sink,
                             recent_window=win)
        got = draft_masks_decode({(0, 0): r}, cfg)[(0, 0)]
        np.testing.assert_array_equal(got, want)


def test_golden_page_aggregate_bit_exact(cuda_ok):
    from paper_2605_15508_b200 import page_aggregate

    g = load_golden("page_aggregate.npz")
    rows = unpack(g["rows"], g["row_offs"])
    outs = unpack(g["out"], g["out_offs"])
    for r, ps, want in zip(rows, g["page_size"], outs):
        got = page_aggregate(r, int(ps))
        assert got.dtype == np.float64
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_golden_verification_masks_c1(cuda_ok):
    from paper_2605_15508_b200 import HeadMapping, SparsityConfig, verification_masks

    g = load_golden("verification_c1.npz")
    entries = {(int(a), int(b)): ((int(c), int(d)), 0) for a, b, c, d in g["entries"]}
    draft_heads = [tuple(map(int, x)) for x in g["draft_heads"]]
    base, gamma = 4096, 4
    for variant in ("token", "ties", "page16", "extras"):
        budget, ps, cur, sink, win = json.loads(str(g[f"{variant}_cfg"]))
        cfg = SparsityConfig(budget=budget, page_size=ps, include_current=cur, include_sink=sink,
                             recent_window=win)
        rows = g[f"{variant}_rows"]
        draft_rows = [{hd: rows[i, j, : base + i + 1] for j, hd in enumerate(draft_heads)} for i in range(gamma)]
        got = verification_masks(draft_rows, base, cfg, HeadMapping(410, entries))
        want = unpack(g[f"{variant}_out"], g[f"{variant}_offs"])
        for t_i, t in enumerate(sorted(got)):
            for i in range(gamma):
                np.testing.assert_array_equal(got[t][i], want[t_i * gamma + i])


def test_golden_prefill(cuda_ok):
    from paper_2605_15508_b200 import SparsityConfig, draft_masks_prefill

    g = load_golden("prefill.npz")
    mats = unpack(g["mats"], g["mat_offs"])
    outs = unpack(g["out"], g["out_offs"])
    j = 0
    for mat, (n, budget, ps) in zip(mats, json.loads(str(g["cfg"]))):
        got = draft_masks_prefill({(0, 0): mat.reshape(n, n)}, SparsityConfig(budget=budget, page_size=ps))[(0, 0)]
        for row in got:
            np.testing.assert_array_equal(row, outs[j])
            j += 1


@pytest.mark.parametrize("kind", ["softmax", "ties", "coarse", "special"])
@pytest.mark.parametrize("ps", [1, 2, 16, 33])
def test_random_rows_vs_oracle(cuda_ok, kind, ps):
    from paper_2605_15508_b200 import SparsityConfig
    from paper_2605_15508_b200.sparsity import select_rows

    rng = np.random.default_rng(hash((kind, ps)) % 2**32)
    for budget, cur, sink, win in ((0.1, True, False, 0), (0.02, False, True, 7), (37, True, True, 64),
                                   (0.5, False, False, 0), (1, False, False, 0)):
        ns = [1, 2, 3, 31, 32, 33, 1023, 1024, 1025, 4097, 20000]
        rows = [_rows_kind(rng, n, kind) for n in ns]
        cfg = SparsityConfig(budget=budget, page_size=ps, include_current=cur, include_sink=sink,
                             recent_window=win)
        got = select_rows(rows, cfg)
        ocfg = O.OracleSparsityConfig(budget, ps, cur, sink, win)
        for r, m in zip(rows, got):
            np.testing.assert_array_equal(m, O.select_row(r, ocfg))


@pytest.mark.parametrize("n", [49152, 49153, 131073])
def test_long_rows_global_key_path(cuda_ok, n):
    """Rows longer than the shared-memory key buffer use the workspace path."""
    from paper_2605_15508_b200 import SparsityConfig
    from paper_2605_15508_b200.sparsity import select_rows

    rng = np.random.default_rng(n)
    rows = [_rows_kind(rng, n, "softmax"), _rows_kind(rng, n, "ties"), _rows_kind(rng, n - 7, "coarse")]
    for ps in (1, 16):
        cfg = SparsityConfig(budget=0.1, page_size=ps)
        got = select_rows(rows, cfg)
        for r, m in zip(rows, got):
            np.testing.assert_array_equal(m, O.select_row(r, O.OracleSparsityConfig(0.1, ps)))


def test_mode_s_head_group_reduction(cuda_ok):
    """row_src sums (fp32, source order) then selects over the committed
    prefix and appends the in-block tail: bit-exact vs the mode-S restatement."""
    import torch

    from paper_2605_15508_b200 import kernels

    rng = np.random.default_rng(7)
    S, n_cols, base, tail = 24, 3000, 2990, 5
    D = np.stack([_rows_kind(rng, n_cols, "softmax") for _ in range(S)])
    D[3] = _rows_kind(rng, n_cols, "ties")
    src = rng.integers(0, S, size=(10, 4)).astype(np.int32)
    src[2] = [3, 3, 3, 3]
    for ps, sink, win in ((1, False, 0), (16, True, 32), (4, False, 100)):
        ocfg = O.OracleSparsityConfig(0.1, ps, False, sink, win)
        b = ocfg.tokens_for_context(base + 1)
        idx, cnt = kernels.select_topk(torch.from_numpy(D).cuda(), row_src=torch.from_numpy(src), n_common=base,
                                       budget=int(b), page_size=ps, include_current=False, include_sink=sink,
                                       recent_window=win, tail_len=tail)
        idx, cnt = idx.cpu().numpy(), cnt.cpu().numpy()
        for r in range(src.shape[0]):
            red = O.reduce_rows_fp32([D[s] for s in src[r]])
            want = O.mode_s_index_list(red, base, tail, ocfg)
            np.testing.assert_array_equal(idx[r, : cnt[r]], want)


def test_capacity_status_flag(cuda_ok):
    import torch

    from paper_2605_15508_b200 import kernels

    x = torch.rand((2, 100), device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    kernels.select_topk(x, budget=50, include_current=False, idx_ld=10, status=status)
    torch.cuda.synchronize()
    assert status.item() & 0x1


@pytest.mark.parametrize("n", [8192, 8193, 16384, 16385, 32767, 32768, 32769, 36864, 36865])
def test_register_select_boundaries(cuda_ok, n):
    """Token rows around the register kernel's capacity steps (8K / 16K / 32K /
    36K keys per CTA; 36865 falls back to select_kernel): every row kind, ties
    spanning many warps (coarse rows), extras — bit-exact vs the oracle."""
    from paper_2605_15508_b200 import SparsityConfig
    from paper_2605_15508_b200.sparsity import select_rows

    rng = np.random.default_rng(n)
    rows = [_rows_kind(rng, n, k) for k in ("softmax", "ties", "coarse", "special")]
    rows.append(_rows_kind(rng, n - 5, "coarse"))  # ragged last warp
    for budget, cur, sink, win in ((0.1, True, False, 0), (0.3, False, True, 300), (4096, True, True, 1)):
        cfg = SparsityConfig(budget=budget, page_size=1, include_current=cur, include_sink=sink,
                             recent_window=win)
        got = select_rows(rows, cfg)
        ocfg = O.OracleSparsityConfig(budget, 1, cur, sink, win)
        for r, m in zip(rows, got):
            np.testing.assert_array_equal(m, O.select_row(r, ocfg))


@pytest.mark.parametrize("nsrc", [1, 2, 3, 4, 5])
def test_register_select_head_groups_32k(cuda_ok, nsrc):
    """Mode-S group sums at the c2 row length (32K committed keys) through the
    register kernel's per-nsrc instances, tie-heavy sources included."""
    import torch

    from paper_2605_15508_b200 import kernels

    rng = np.random.default_rng(100 + nsrc)
    S, base, tail = 12, 32768, 5
    D = np.stack([_rows_kind(rng, base + tail, "softmax" if s % 3 else "coarse") for s in range(S)])
    src = rng.integers(0, S, size=(6, nsrc)).astype(np.int32)
    ocfg = O.OracleSparsityConfig(0.1, 1, False, False, 0)
    b = ocfg.tokens_for_context(base + 1)
    idx, cnt = kernels.select_topk(torch.from_numpy(D).cuda(), row_src=torch.from_numpy(src), n_common=base,
                                   budget=int(b), page_size=1, include_current=False, tail_len=tail)
    idx, cnt = idx.cpu().numpy(), cnt.cpu().numpy()
    for r in range(src.shape[0]):
        red = O.reduce_rows_fp32([D[s] for s in src[r]])
        np.testing.assert_array_equal(idx[r, : cnt[r]], O.mode_s_index_list(red, base, tail, ocfg))
