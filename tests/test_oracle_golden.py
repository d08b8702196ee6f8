"""Pin the CPU oracle against the reference's golden vectors (CPU only).

The vectors were produced by running the real reference package
(tests/golden/make_golden.py). The known-answer cases are copied from the
reference's own tests (pkg/tests/test_numkit.py:86-113,
pkg/tests/test_sparsity.py:31-235).
"""

import json
import math

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from conftest import cfg_from_json, load_golden, unpack
from oracle import sts_oracle as O


# ---- reference known-answer tests ---------------------------------------------


def test_topk_known_answers():
    # pkg/tests/test_numkit.py:86-93
    assert list(O.topk_indices([0.1, 0.7, 0.2], 2)) == [1, 2]
    assert list(O.topk_indices([0.5, 0.5, 0.5], 1)) == [0]
    assert list(O.topk_indices([3.0, 1.0, 2.0], 10)) == [0, 1, 2]
    with pytest.raises(O.OracleContractViolation):
        O.topk_indices([], 1)
    with pytest.raises(O.OracleContractViolation):
        O.topk_indices([1.0], 0)


@settings(max_examples=200, deadline=None)
@given(st.lists(st.floats(-1, 1, allow_nan=False), min_size=1, max_size=64), st.integers(1, 64))
def test_topk_brute_force(scores, k):
    # pkg/tests/test_numkit.py:103-113
    got = O.topk_indices(scores, k)
    ranked = sorted(range(len(scores)), key=lambda i: (-scores[i], i))
    assert list(got) == sorted(ranked[: min(k, len(scores))])


def test_page_aggregate_known_answers():
    # pkg/tests/test_sparsity.py:31-44
    np.testing.assert_allclose(O.page_aggregate([0.2, 0.5, 0.3], 1), [0.2, 0.5, 0.3])
    np.testing.assert_allclose(O.page_aggregate([0.05, 0.6, 0.05, 0.3], 2), [0.65, 0.35])
    np.testing.assert_allclose(O.page_aggregate(np.ones(5), 2), [2.0, 2.0, 1.0])


def test_decode_mask_known_answers():
    # pkg/tests/test_sparsity.py:47-82
    C = O.OracleSparsityConfig
    row = np.array([0.05, 0.6, 0.05, 0.3])
    assert list(O.select_row(row, C(2))) == [1, 3]
    assert list(O.select_row(np.array([0.4, 0.3, 0.2, 0.1]), C(2, include_current=False))) == [0, 1]
    assert list(O.select_row(np.array([0.4, 0.3, 0.2, 0.1]), C(2))) == [0, 1, 3]
    assert list(O.select_row(row, C(2, page_size=2))) == [0, 1, 3]
    assert list(O.select_row(row, C(99))) == [0, 1, 2, 3]
    assert O.select_row(np.linspace(1.0, 0.1, 10), C(1 / 8, include_current=False)).size == 2
    assert list(O.select_row(np.array([0.0, 0.0, 0.9, 0.05, 0.05]), C(1, include_sink=True, recent_window=2))) == [0, 2, 3, 4]


def test_sparse_attention_known_answers():
    # pkg/tests/test_sparsity.py:209-235
    rng = np.random.default_rng(3)
    q, k, v = rng.standard_normal(6), rng.standard_normal((10, 6)), rng.standard_normal((10, 6))
    np.testing.assert_allclose(O.sparse_attention(q, k, v, np.array([4])), v[4], rtol=1e-6)
    with pytest.raises(O.OracleContractViolation):
        O.sparse_attention(q, k, v, np.array([], dtype=np.int64))
    with pytest.raises(O.OracleContractViolation):
        O.sparse_attention(q, k, v, np.array([10]))


# ---- golden vectors from the real reference --------------------------------------


def test_golden_topk():
    g = load_golden("topk.npz")
    rows = unpack(g["rows"], g["row_offs"])
    outs = unpack(g["out"], g["out_offs"])
    for r, k, want in zip(rows, g["k"], outs):
        np.testing.assert_array_equal(O.topk_indices(r, int(k)), want)


def test_golden_page_aggregate_and_pairwise_order():
    g = load_golden("page_aggregate.npz")
    rows = unpack(g["rows"], g["row_offs"])
    outs = unpack(g["out"], g["out_offs"])
    for r, ps, want in zip(rows, g["page_size"], outs):
        got = O.page_aggregate(r, int(ps))
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64))  # bit-exact
        # explicit pairwise restatement (the order the CUDA kernel uses)
        x = r.astype(np.float64)
        ps = int(ps)
        mine = [x[p] + O.numpy_pairwise_sum(x[p + 1 : min(p + ps, x.size)]) if ps > 1 else x[p]
                for p in range(0, x.size, ps)]
        assert np.array_equal(np.asarray(mine, np.float64).view(np.uint64), want.view(np.uint64))


def test_golden_select_row():
    g = load_golden("select_row.npz")
    rows = unpack(g["rows"], g["row_offs"])
    outs = unpack(g["out"], g["out_offs"])
    for r, c, want in zip(rows, json.loads(str(g["cfg"])), outs):
        budget, ps, cur, sink, win = cfg_from_json(c)
        cfg = O.OracleSparsityConfig(budget, ps, cur, sink, win)
        np.testing.assert_array_equal(O.select_row(r, cfg), want)


def test_golden_verification_masks_c1():
    g = load_golden("verification_c1.npz")
    entries = {(int(a), int(b)): ((int(c), int(d)), 0) for a, b, c, d in g["entries"]}
    draft_heads = [tuple(map(int, x)) for x in g["draft_heads"]]
    base, gamma = 4096, 4
    for variant in ("token", "ties", "page16", "extras"):
        budget, ps, cur, sink, win = json.loads(str(g[f"{variant}_cfg"]))
        cfg = O.OracleSparsityConfig(budget, ps, cur, sink, win)
        rows = g[f"{variant}_rows"]
        draft_rows = [{hd: rows[i, j, : base + i + 1] for j, hd in enumerate(draft_heads)} for i in range(gamma)]
        got = O.verification_masks(draft_rows, base, cfg, entries)
        want = unpack(g[f"{variant}_out"], g[f"{variant}_offs"])
        for t_i, t in enumerate(sorted(got)):
            for i in range(gamma):
                np.testing.assert_array_equal(got[t][i], want[t_i * gamma + i])


def test_golden_prefill():
    g = load_golden("prefill.npz")
    mats = unpack(g["mats"], g["mat_offs"])
    outs = unpack(g["out"], g["out_offs"])
    j = 0
    for mat, (n, budget, ps) in zip(mats, json.loads(str(g["cfg"]))):
        mat = mat.reshape(n, n)
        got = O.draft_masks_prefill({(0, 0): mat}, O.OracleSparsityConfig(budget, ps))[(0, 0)]
        for row in got:
            np.testing.assert_array_equal(row, outs[j])
            j += 1


def test_golden_sparse_attention():
    g = load_golden("sparse_attention.npz")
    qo = ko = mo = oo = 0
    masks = unpack(g["mask"], g["mask_offs"])
    for (n, d), mask in zip(g["shapes"], masks):
        q = g["q"][qo : qo + d]; qo += d
        k = g["k"][ko : ko + n * d].reshape(n, d)
        v = g["v"][ko : ko + n * d].reshape(n, d); ko += n * d
        want = g["out"][oo : oo + d]; oo += d
        got = O.sparse_attention(q, k, v, mask)
        np.testing.assert_array_equal(got, want)  # same fp64 ops -> identical
        out2, _ = O.block_attention(q[None], k, v, mask)
        np.testing.assert_allclose(out2[0], want, rtol=1e-5, atol=1e-6)


def test_golden_capture_rows():
    g = load_golden("capture.npz")
    base = int(g["base"])
    keys0, q0, rows = g["keys0"], g["q0"], g["rows"]
    H = q0.shape[1]
    for i in range(q0.shape[0]):
        for h in range(H):
            got = O.draft_attention_rows(q0[i, h][None], keys0[:, h, :], base + i, 1)[0]
            want = rows[i, h, : base + i + 1]
            np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-7)


# ---- restatement self-consistency (new semantics) ---------------------------------


def test_fp32_order_keys_rank_like_reference():
    rng = np.random.default_rng(0)
    x = rng.standard_normal(500).astype(np.float32)
    x[::17] = np.nan
    x[::23] = -0.0
    x[::29] = 0.0
    x[::31] = np.inf
    x[::37] = -np.inf
    keys = O.fp32_order_keys(x)
    order = sorted(range(x.size), key=lambda i: (-int(keys[i]), i))
    for k in (1, 7, 100, 499, 500):
        np.testing.assert_array_equal(np.sort(order[:k]), O.topk_indices(x, k))


def test_sharded_threshold_equals_global_topk():
    rng = np.random.default_rng(1)
    for trial in range(20):
        n = int(rng.integers(50, 3000))
        x = (np.round(rng.random(n) * 64) / 64).astype(np.float32)  # tie-heavy
        k = int(rng.integers(1, n))
        nr = int(rng.integers(1, 9))
        bounds = O.shard_bounds(n, nr)
        keys = O.fp32_order_keys(x)
        # global threshold from summed histograms == kth largest key
        T = np.sort(keys)[::-1][k - 1]
        gt = [int((keys[lo:hi] > T).sum()) for lo, hi in bounds]
        ties = [int((keys[lo:hi] == T).sum()) for lo, hi in bounds]
        need = k - sum(gt)
        sel = []
        before = 0
        for (lo, hi), t in zip(bounds, ties):
            take = min(max(need - before, 0), t)
            before += t
            tie_pos = np.nonzero(keys[lo:hi] == T)[0][:take]
            sel.extend((lo + np.nonzero(keys[lo:hi] > T)[0]).tolist())
            sel.extend((lo + tie_pos).tolist())
        np.testing.assert_array_equal(np.sort(sel), O.topk_indices(x, k))


def test_lse_merge_equals_union_attention():
    rng = np.random.default_rng(2)
    n, d = 400, 32
    q = rng.standard_normal(d)
    k = rng.standard_normal((n, d))
    v = rng.standard_normal((n, d))
    mask = np.sort(rng.choice(n, 120, replace=False))
    want = O.sparse_attention(q, k, v, mask)
    outs, lses = [], []
    for lo, hi in O.shard_bounds(n, 4):
        m = mask[(mask >= lo) & (mask < hi)]
        o, l = O.sparse_attention_lse(q, k, v, m)
        outs.append(o[None]); lses.append(np.array([l]))
    merged, _ = O.lse_merge(outs, lses)
    np.testing.assert_allclose(merged[0], want, rtol=1e-5, atol=1e-6)


def test_lru_prefetch_matches_reference_simulator():
    """The resident-pool restatement reproduces the reference simulator's
    per-step transfers (specsparse.offloadsim.simulate('prefetch'), recorded
    by tests/golden/make_offload_golden.py)."""
    import json
    from pathlib import Path

    from oracle import sts_oracle as O

    g = json.loads((Path(__file__).resolve().parent / "golden" / "offload_lru.json").read_text())
    for case in g["cases"]:
        missing = O.lru_prefetch_steps(case["traces"], case["capacity"])
        assert [len(m) for m in missing] == case["missing_per_step"]
