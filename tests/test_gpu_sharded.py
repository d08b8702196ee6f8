"""GPU parity of the sequence-sharded path on one B200.

P virtual ranks run the real sharded kernels on P shards of one GPU's
tensors, their collectives serviced in-process (sharded.run_lockstep).  The
bar: the union of the ranks' selections equals the single-GPU selection of the
concatenated row BIT-EXACTLY (ties to the lowest global index), and equals the
oracle; the LSE-merged attention matches the oracle within the bf16 tolerance.
"""

import numpy as np
import pytest

from oracle import sts_oracle as O
from test_gpu_select import _rows_kind

pytestmark = pytest.mark.gpu


def _dist_select(scores, row_src, n_global, k_top, P, ps=1, sink=False, win=0, cur=False, tail=0, n_kv=None):
    import torch

    from paper_2605_15508_b200 import sharded

    n_kv = n_global + tail if n_kv is None else n_kv
    bounds = sharded.shard_bounds(n_kv, P, ps)
    rows = row_src.shape[0] if row_src is not None else scores.shape[0]
    gens, outs = [], []
    for r, (lo, hi) in enumerate(bounds):
        n_loc = hi - lo
        sel = sharded.DistSelector(rows, n_loc, ps, P, scores.device)
        idx = torch.full((rows, max(n_loc, 1)), -1, dtype=torch.int32, device=scores.device)
        cnt = torch.zeros((rows,), dtype=torch.int32, device=scores.device)
        view = scores[:, lo:hi] if n_loc > 0 else scores[:, :1]
        gens.append(sel.protocol(view, row_src=row_src, n_global=n_global, lo=lo, k_top=k_top, rank=r,
                                 include_current=cur, include_sink=sink, recent_window=win, tail_len=tail,
                                 n_kv_local=n_loc, idx=idx, cnt=cnt))
        outs.append((lo, idx, cnt, sel))
    sharded.run_lockstep(gens)
    torch.cuda.synchronize()
    merged = []
    for row in range(rows):
        parts = []
        for lo, idx, cnt, _ in outs:
            c = int(cnt[row])
            parts.append(lo + idx[row, :c].cpu().numpy().astype(np.int64))
        merged.append(np.concatenate(parts))
    return merged


@pytest.mark.parametrize("kind", ["softmax", "ties", "coarse"])
@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_dist_select_equals_single_gpu_select(cuda_ok, kind, P):
    import torch

    from paper_2605_15508_b200 import kernels

    rng = np.random.default_rng(P * 7 + len(kind))
    n, rows = 5000, 6
    x = np.stack([_rows_kind(rng, n, kind) for _ in range(rows)])
    scores = torch.from_numpy(x).cuda()
    for k in (1, 37, 500, 4999, 5000, 6000):
        got = _dist_select(scores, None, n, k, P)
        idx, cnt = kernels.select_topk(scores, budget=k, include_current=False, n_common=n)
        for r in range(rows):
            want = idx[r, : int(cnt[r])].cpu().numpy()
            assert np.array_equal(got[r], want), (kind, P, k, r)
            assert np.array_equal(got[r], O.topk_indices(x[r], k) if k < n else np.arange(n))


@pytest.mark.parametrize("P", [2, 5])
def test_dist_select_head_group_sum_extras_and_tail(cuda_ok, P):
    """Mode-S rows (fp32 sum of 4 mapped source rows), sink + recent window,
    in-block tail of 5 positions, budget from the fraction rule."""
    import torch

    from paper_2605_15508_b200 import kernels

    rng = np.random.default_rng(11 + P)
    n, S, rows, tail = 3001, 12, 9, 5
    x = np.stack([_rows_kind(rng, n + tail + 3, "ties") for _ in range(S)])
    scores = torch.from_numpy(x).cuda()
    src = torch.from_numpy(rng.integers(0, S, (rows, 4)).astype(np.int32)).cuda()
    k = 301
    got = _dist_select(scores, src, n, k, P, sink=True, win=17, tail=tail)
    idx, cnt = kernels.select_topk(scores, row_src=src, budget=k, include_current=False, include_sink=True,
                                   recent_window=17, n_common=n, tail_len=tail)
    cfg = O.OracleSparsityConfig(0.1, 1, False, True, 17)
    for r in range(rows):
        want = idx[r, : int(cnt[r])].cpu().numpy()
        assert np.array_equal(got[r], want), (P, r)
        red = O.reduce_rows_fp32([x[j] for j in src[r].cpu().numpy()])
        sel = O.select_committed(red, n, k, cfg)
        assert np.array_equal(got[r], np.concatenate([sel, np.arange(n, n + tail)]))


@pytest.mark.parametrize("ps,P", [(4, 3), (16, 4)])
def test_dist_select_page_mode(cuda_ok, ps, P):
    import torch

    from paper_2605_15508_b200 import kernels

    rng = np.random.default_rng(ps + P)
    n, rows = 4099, 5
    x = np.stack([_rows_kind(rng, n, "ties") for _ in range(rows)])
    scores = torch.from_numpy(x).cuda()
    for b in (1, 50, 410, 4098):
        kp = -(-b // ps)
        got = _dist_select(scores, None, n, kp, P, ps=ps)
        idx, cnt = kernels.select_topk(scores, budget=b, page_size=ps, include_current=False, n_common=n)
        for r in range(rows):
            want = idx[r, : int(cnt[r])].cpu().numpy()
            assert np.array_equal(got[r], want), (ps, P, b, r)


def test_sharded_verify_step_matches_oracle(cuda_ok):
    import torch

    from paper_2605_15508_b200 import SparsityConfig, kernels, sharded
    from paper_2605_15508_b200.verify_step import VerifyShape, random_mapping_table, synthetic_inputs

    s = VerifyShape(batch=1, context=3000, gamma=4, target_layers=2, target_q_heads=8, target_kv_heads=2,
                    head_dim=128, draft_layers=2, draft_q_heads=8, draft_kv_heads=2, draft_head_dim=64)
    cfg = SparsityConfig(budget=0.1)
    table = random_mapping_table(s, seed=3)
    P = 3
    dq, dk, tq, tk, tv = synthetic_inputs(s, "cuda", seed=7)
    steps = [sharded.ShardedVerifyStep(s, cfg, table, r, P, device="cuda") for r in range(P)]
    views = [st.local_views(dq, dk, tq, tk, tv) for st in steps]
    outs = sharded.run_lockstep([st.step(*v) for st, v in zip(steps, views)])
    torch.cuda.synchronize()
    assert all(int(st.status.item()) == 0 for st in steps)
    # every rank ends with the same merged output
    for o, _ in outs[1:]:
        assert torch.equal(o, outs[0][0])
    # concatenated draft rows -> oracle mode-S masks, bit-exact
    D = np.concatenate([st.draft_rows[:, : st.n_loc].cpu().numpy() for st in steps], axis=1)
    src = steps[0].row_src.cpu().numpy()
    ocfg = O.OracleSparsityConfig(0.1, 1, False, False, 0)
    qf = tq.reshape(s.target_units, -1, s.head_dim).float().cpu().numpy()
    kf = tk.flatten(0, 2).float().cpu().numpy()
    vf = tv.flatten(0, 2).float().cpu().numpy()
    out = outs[0][0].float().cpu().numpy()
    for u in range(s.target_units):
        want_idx = O.mode_s_index_list(O.reduce_rows_fp32([D[j] for j in src[u]]), s.context, s.rows, ocfg)
        got_idx = np.concatenate([st.lo + st.idx[u, : int(st.cnt[u])].cpu().numpy() for st in steps])
        assert np.array_equal(got_idx, want_idx), u
        want, _ = O.block_attention(qf[u], kf[u], vf[u], want_idx, causal_base=s.context, rows_per_head=s.rows)
        np.testing.assert_allclose(out[u], want, rtol=2e-2, atol=2e-2)
    # the sharded capture's rows match the single-GPU capture within fp32 ulps
    one = sharded.ShardedVerifyStep(s, cfg, table, 0, 1, device="cuda")
    sharded.run_single(one.capture(*one.local_views(dq, dk, tq, tk, tv)[:2]))
    np.testing.assert_allclose(D, one.draft_rows[:, : s.n_kv].cpu().numpy(), rtol=1e-5, atol=1e-9)
    # dense sharded baseline == dense single-GPU decode
    dense = sharded.run_lockstep([st.attend_dense(*v[2:]) for st, v in zip(steps, views)])
    q1, k1, v1 = tq.reshape(s.target_units, -1, s.head_dim), tk.flatten(0, 2), tv.flatten(0, 2)
    ref, _ = kernels.sparse_decode(q1, k1, v1, n_dense=s.n_kv, causal_base=s.context, rows_per_head=s.rows)
    np.testing.assert_allclose(dense[0][0].float().cpu().numpy(), ref.float().cpu().numpy(), rtol=2e-2, atol=2e-2)


def test_p2p_merge_matches_gather_merge(cuda_ok):
    """The peer-pointer merge (sts_lse_merge_ptrs: every rank's partial read
    through a device array of pointers, as over NVLink symmetric memory) gives
    the all-gather + merge result bit for bit (virtual ranks on one GPU)."""
    import torch

    from paper_2605_15508_b200 import SparsityConfig, sharded
    from paper_2605_15508_b200.verify_step import VerifyShape, random_mapping_table, synthetic_inputs

    s = VerifyShape(batch=1, context=2500, gamma=4, target_layers=2, target_q_heads=8, target_kv_heads=2,
                    head_dim=128, draft_layers=2, draft_q_heads=8, draft_kv_heads=2, draft_head_dim=64)
    cfg = SparsityConfig(budget=0.1)
    table = random_mapping_table(s, seed=4)
    dq, dk, tq, tk, tv = synthetic_inputs(s, "cuda", seed=9)
    P = 3
    outs = {}
    for mode in ("gather", "p2p"):
        steps = [sharded.ShardedVerifyStep(s, cfg, table, r, P, device="cuda") for r in range(P)]
        if mode == "p2p":
            keep = sharded.link_p2p_lockstep(steps)  # noqa: F841 (buffers stay alive)
        views = [st.local_views(dq, dk, tq, tk, tv) for st in steps]
        res = sharded.run_lockstep([st.step(*v) for st, v in zip(steps, views)])
        torch.cuda.synchronize()
        outs[mode] = [o.clone() for o, _ in res]
    for a, b in zip(outs["gather"], outs["p2p"]):
        assert torch.equal(a, b)


def test_heads_times_sequence_sharding(cuda_ok):
    """BASELINE config 5's layout: 2 head groups x 2 sequence shards (4 virtual
    ranks). Each head group runs its own sequence-sharded protocol over its
    kv-heads; together they reproduce the single-GPU masks and attention."""
    import torch

    from paper_2605_15508_b200 import SparsityConfig, sharded
    from paper_2605_15508_b200.verify_step import VerifyShape, random_mapping_table, synthetic_inputs

    s = VerifyShape(batch=2, context=1800, gamma=4, target_layers=2, target_q_heads=8, target_kv_heads=4,
                    head_dim=128, draft_layers=2, draft_q_heads=8, draft_kv_heads=2, draft_head_dim=64)
    cfg = SparsityConfig(budget=0.1)
    table = random_mapping_table(s, seed=6)
    dq, dk, tq, tk, tv = synthetic_inputs(s, "cuda", seed=12)
    hp, sp = 2, 2
    qf = tq.reshape(s.batch, s.target_layers, s.target_kv_heads, -1, s.head_dim).float().cpu().numpy()
    kf = tk.float().cpu().numpy()
    vf = tv.float().cpu().numpy()
    ocfg = O.OracleSparsityConfig(0.1, 1, False, False, 0)
    for g in range(hp):
        steps = [sharded.ShardedVerifyStep(s, cfg, table, r, sp, device="cuda", head_groups=hp, head_group=g)
                 for r in range(sp)]
        views = [st.local_views(dq, dk, tq, tk, tv) for st in steps]
        outs = sharded.run_lockstep([st.step(*v) for st, v in zip(steps, views)])
        torch.cuda.synchronize()
        D = np.concatenate([st.draft_rows[:, : st.n_loc].cpu().numpy() for st in steps], axis=1)
        src = steps[0].row_src.cpu().numpy()
        out = outs[0][0].float().cpu().numpy()
        hkv = s.target_kv_heads // hp
        for u in range(steps[0].U):
            b, rest = divmod(u, s.target_layers * hkv)
            l, h = divmod(rest, hkv)
            kvh = g * hkv + h
            want_idx = O.mode_s_index_list(O.reduce_rows_fp32([D[j] for j in src[u]]), s.context, s.rows, ocfg)
            got_idx = np.concatenate([st.lo + st.idx[u, : int(st.cnt[u])].cpu().numpy() for st in steps])
            assert np.array_equal(got_idx, want_idx), (g, u)
            want, _ = O.block_attention(qf[b, l, kvh], kf[b, l, kvh], vf[b, l, kvh], want_idx,
                                        causal_base=s.context, rows_per_head=s.rows)
            np.testing.assert_allclose(out[u], want, rtol=2e-2, atol=2e-2)


@pytest.mark.parametrize("ps", [1, 16])
@pytest.mark.parametrize("P", [1, 3])
def test_dist_select_long_rows_span_chunks(cuda_ok, ps, P):
    """Rows longer than two CTA chunks of every sharded-select pass (key and
    histogram passes: 32768 positions per CTA; emit: 16384): the cross-CTA
    histogram atomics, the per-chunk tie prefix of the bits pass and the
    token-count prefix of the write pass all run.  Tie-heavy mode-S rows
    (4 summed sources), sink + recent window + in-block tail; bit-exact vs
    the single-CTA select_kernel and the oracle."""
    import torch

    from paper_2605_15508_b200 import kernels

    rng = np.random.default_rng(70001 + ps + P)
    n, S, rows, tail = 70001, 6, 4, 5
    x = np.stack([_rows_kind(rng, n + tail + 3, "ties") for _ in range(S)])
    scores = torch.from_numpy(x).cuda()
    src = torch.from_numpy(rng.integers(0, S, (rows, 4)).astype(np.int32)).cuda()
    b = 7001
    kp = b if ps == 1 else -(-b // ps)
    got = _dist_select(scores, src, n, kp, P, ps=ps, sink=True, win=33, tail=tail)
    idx, cnt = kernels.select_topk(scores, row_src=src, budget=b, page_size=ps, include_current=False,
                                   include_sink=True, recent_window=33, n_common=n, tail_len=tail)
    cfg = O.OracleSparsityConfig(0.1, ps, False, True, 33)
    for r in range(rows):
        want = idx[r, : int(cnt[r])].cpu().numpy()
        assert np.array_equal(got[r], want), (ps, P, r)
        red = O.reduce_rows_fp32([x[j] for j in src[r].cpu().numpy()])
        sel = O.select_committed(red, n, b, cfg)
        assert np.array_equal(got[r], np.concatenate([sel, np.arange(n, n + tail)]))


def test_two_process_sharded_step_parity(cuda_ok, tmp_path):
    """ShardedVerifyStep in two processes (torch.distributed, gloo, both ranks
    on cuda:0): bench.py's N=2 path end to end — local capture, the
    histogram all-reduce rounds, tie-count all-gather, attention and the LSE
    merge — with its sampled-unit oracle check (masks bit-exact, outputs
    within 2e-2)."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    cmd = [sys.executable, str(root / "bench.py"), "--gpus", "2", "--one-gpu", "--dist-backend", "gloo",
           "--context", "65536", "--steps", "1", "--warmup", "3", "--no-single-ref", "--parity-units", "8"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=str(root))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2
    assert line["parity"]["masks_bit_exact"] and line["parity"]["attention_ok"], line["parity"]
