"""GPU parity of draft-score capture and of the full verify step.

Draft scores: the GPU's expf differs from numpy's in the last ulp, so score
rows are checked by tolerance (rtol 1e-3 on bf16 inputs: the fp32 probability
rows vs the fp64 reference math on the same bf16-rounded q/K), and mask
parity is asserted bit-exactly on the GPU-produced rows (SURVEY §7.3 hard
part 1: "selection is bit-exact given identical fp32 score rows").
"""

import numpy as np
import pytest

from oracle import sts_oracle as O

pytestmark = pytest.mark.gpu


def _small_shape(**kw):
    from paper_2605_15508_b200.verify_step import VerifyShape

    d = dict(batch=2, context=1500, gamma=4, target_layers=3, target_q_heads=8, target_kv_heads=2, head_dim=128,
             draft_layers=2, draft_q_heads=8, draft_kv_heads=2, draft_head_dim=64)
    d.update(kw)
    return VerifyShape(**d)


def test_draft_capture_rows_match_reference_math(cuda_ok):
    import torch

    from paper_2605_15508_b200 import kernels

    rng = np.random.default_rng(0)
    U, G, R, d, base = 3, 4, 5, 64, 900
    N = base + R
    q = torch.from_numpy(rng.standard_normal((U, G * R, d)).astype(np.float32)).bfloat16().cuda()
    k = torch.from_numpy(rng.standard_normal((U, N, d)).astype(np.float32)).bfloat16().cuda()
    lse = kernels.draft_lse(q, k, G=G, R=R, base=base)
    rows_r = kernels.draft_probs(q, k, lse, G=G, R=R, base=base, mode="R").cpu().numpy()
    rows_s = kernels.draft_probs(q, k, lse, G=G, R=R, base=base, mode="S").cpu().numpy()
    qf, kf = q.float().cpu().numpy(), k.float().cpu().numpy()
    for u in range(U):
        for hh in range(G):
            ref_rows = O.draft_attention_rows(qf[u, hh * R : (hh + 1) * R], kf[u], base, R)
            for i in range(R):
                got = rows_r[(u * G + hh) * R + i, : base + i + 1]
                np.testing.assert_allclose(got, ref_rows[i], rtol=1e-3, atol=1e-7)
            red = sum(r[:base].astype(np.float64) for r in ref_rows)
            np.testing.assert_allclose(rows_s[u * G + hh, :base], red, rtol=1e-3, atol=1e-7)
            # the GPU's mode-S row is exactly the fp32 sequential sum of its mode-R rows
            mine = O.reduce_rows_fp32([rows_r[(u * G + hh) * R + i, :base] for i in range(R)])
            np.testing.assert_array_equal(rows_s[u * G + hh, :base], mine)


def test_draft_raw_scores_match_reference_math(cuda_ok):
    """sts_draft_scores = the reference's ForwardRecord.scores (raw q.k/sqrt(d)
    per speculative row over its causal prefix; src/toymodel.py:225-240,
    :351-352) on the same bf16-rounded q/K, and softmax of it = the captured
    probabilities."""
    import torch

    from paper_2605_15508_b200 import kernels

    rng = np.random.default_rng(7)
    U, G, R, d, base = 2, 4, 5, 64, 700
    N = base + R
    q = torch.from_numpy(rng.standard_normal((U, G * R, d)).astype(np.float32)).bfloat16().cuda()
    k = torch.from_numpy(rng.standard_normal((U, N, d)).astype(np.float32)).bfloat16().cuda()
    raw = kernels.draft_scores(q, k, G=G, R=R, base=base).cpu().numpy()
    lse = kernels.draft_lse(q, k, G=G, R=R, base=base)
    probs = kernels.draft_probs(q, k, lse, G=G, R=R, base=base, mode="R").cpu().numpy()
    qf, kf = q.double().cpu().numpy(), k.double().cpu().numpy()
    for u in range(U):
        for m in range(G * R):
            i = m % R
            row = (u * G * R) + m
            want = kf[u, : base + i + 1] @ qf[u, m] / np.sqrt(d)
            np.testing.assert_allclose(raw[row, : base + i + 1], want, rtol=1e-4, atol=1e-4)
            assert not raw[row, base + i + 1 :].any()  # beyond the row's prefix: untouched
            sm = np.exp(want - want.max())
            np.testing.assert_allclose(probs[row, : base + i + 1], sm / sm.sum(), rtol=1e-3, atol=1e-7)


@pytest.mark.parametrize("ps,sink,win,long_rows", [(1, False, 0, False), (16, True, 64, False), (1, False, 0, True),
                                                   (16, True, 64, True), (1, True, 32, True)])
def test_verify_step_mode_s(cuda_ok, ps, sink, win, long_rows):
    import torch

    from paper_2605_15508_b200 import SparsityConfig
    from paper_2605_15508_b200.verify_step import STSVerifyStep, random_mapping_table, synthetic_inputs

    s = _small_shape()
    cfg = SparsityConfig(budget=0.1, page_size=ps, include_sink=sink, recent_window=win)
    table = random_mapping_table(s, seed=1)
    # long_rows: the chunk-parallel (sharded-path, P = 1) select instead of one CTA per row
    step = STSVerifyStep(s, cfg, table, mode="S", long_row_min=1 if long_rows else None)
    assert (step._dist is not None) == long_rows
    dq, dk, tq, tk, tv = synthetic_inputs(s, "cuda", seed=3)
    q, k, v = step.target_views(tq, tk, tv)
    dqv, dkv = step.draft_views(dq, dk)
    out, lse = step.step(dqv, dkv, q, k, v)
    torch.cuda.synchronize()
    assert step.status.item() == 0
    D = step.draft_rows.cpu().numpy()
    src = step.row_src.cpu().numpy()
    idx, cnt = step.idx.cpu().numpy(), step.cnt.cpu().numpy()
    ocfg = O.OracleSparsityConfig(0.1, ps, False, sink, win)
    qf, kf, vf = q.float().cpu().numpy(), k.float().cpu().numpy(), v.float().cpu().numpy()
    out = out.float().cpu().numpy()
    for u in range(s.target_units):
        red = O.reduce_rows_fp32([D[j] for j in src[u]])
        want_idx = O.mode_s_index_list(red, s.context, s.rows, ocfg)
        np.testing.assert_array_equal(idx[u, : cnt[u]], want_idx)  # bit-exact masks
        want, _ = O.block_attention(qf[u], kf[u], vf[u], want_idx, causal_base=s.context, rows_per_head=s.rows)
        np.testing.assert_allclose(out[u], want, rtol=2e-2, atol=2e-2)


def test_verify_step_mode_r_reference_masks(cuda_ok):
    """Mode R reproduces the reference's per-(head,row) verification masks
    (specdec._verification_masks) on the GPU-captured rows, under GQA."""
    import torch

    from paper_2605_15508_b200 import SparsityConfig
    from paper_2605_15508_b200.verify_step import STSVerifyStep, random_mapping_table, synthetic_inputs

    s = _small_shape(batch=1)
    cfg = SparsityConfig(budget=0.1)
    table = random_mapping_table(s, seed=2)
    step = STSVerifyStep(s, cfg, table, mode="R")
    dq, dk, tq, tk, tv = synthetic_inputs(s, "cuda", seed=4)
    q, k, v = step.target_views(tq, tk, tv)
    dqv, dkv = step.draft_views(dq, dk)
    out, _ = step.step(dqv, dkv, q, k, v)
    torch.cuda.synchronize()
    assert step.status.item() == 0
    P = step.draft_rows.cpu().numpy()
    R, base, Gt = s.rows, s.context, s.target_group
    nd = s.draft_layers * s.draft_q_heads
    # reference wiring on the GPU-captured rows
    draft_heads = [(dl, dh) for dl in range(s.draft_layers) for dh in range(s.draft_q_heads)]
    draft_rows = [{hd: P[(j) * R + i, : base + i + 1] for j, hd in enumerate(draft_heads)} for i in range(R)]
    entries = {(l, h): (draft_heads[int(table[l, h])], 0) for l in range(s.target_layers) for h in range(s.target_q_heads)}
    ref = O.verification_masks(draft_rows, base, O.OracleSparsityConfig(0.1), entries)
    qf, kf, vf = q.float().cpu().numpy(), k.float().cpu().numpy(), v.float().cpu().numpy()
    out = out.float().cpu().numpy()
    idx, mem, cnt = step.idx.cpu().numpy(), step.member.cpu().numpy().view(np.uint32), step.cnt.cpu().numpy()
    for l in range(s.target_layers):
        for g in range(s.target_kv_heads):
            u = l * s.target_kv_heads + g
            lst = idx[u, : cnt[u]]
            for hh in range(Gt):
                for i in range(R):
                    r = hh * R + i
                    mask = ref[(l, g * Gt + hh)][i]
                    np.testing.assert_array_equal(lst[(mem[u, : cnt[u]] >> r) & 1 == 1], mask)
                    want = O.sparse_attention(qf[u, r], kf[u], vf[u], mask)
                    np.testing.assert_allclose(out[u, r], want, rtol=2e-2, atol=2e-2)


def test_host_buffer_api_matches_device_path(cuda_ok):
    """STSVerifyStep.step_host / attend_host (pinned host queries in, host output
    out, CUDA-graph replays) give the device path's result bit for bit."""
    import torch

    from paper_2605_15508_b200 import SparsityConfig
    from paper_2605_15508_b200.verify_step import STSVerifyStep, random_mapping_table, synthetic_inputs

    s = _small_shape()
    step = STSVerifyStep(s, SparsityConfig(budget=0.1), random_mapping_table(s, seed=2), mode="S")
    dq, dk, tq, tk, tv = synthetic_inputs(s, "cuda", seed=3)
    q, k, v = step.target_views(tq, tk, tv)
    out, _ = step.step(*step.draft_views(dq, dk), q, k, v)
    want = out.clone()
    h_out = torch.empty(want.shape, dtype=want.dtype).pin_memory()
    for _ in range(2):  # first call captures the graph, second replays it
        h_out.zero_()
        step.step_host(dq.cpu().pin_memory(), dk, tq.cpu().pin_memory(), tk, tv, h_out, chunks=1)
        torch.cuda.synchronize()
        assert torch.equal(h_out, want.cpu())
    # default: the kernel writes the pinned output directly (one launch); and
    # the copy-engine form (D2H after the kernel)
    for kw in ({}, {"direct_out": False, "chunks": 1}):
        for _ in range(2):
            h_out.zero_()
            step.attend_host(tq.cpu().pin_memory(), tk, tv, h_out, **kw)
            torch.cuda.synchronize()
            assert torch.equal(h_out, want.cpu()), kw
    # a pinned output of another shape with the same elements (flat): direct
    h_flat = torch.empty(want.numel(), dtype=want.dtype).pin_memory()
    step.attend_host(tq.cpu().pin_memory(), tk, tv, h_flat)
    torch.cuda.synchronize()
    assert torch.equal(h_flat.view(want.shape), want.cpu())
    # units in C groups (pipelined copies or direct writes; per-group work
    # splits differ, so the fp32 merge order may differ from the one-launch
    # run: tolerance)
    h_tq = tq.cpu().pin_memory()
    for C in (2, 3):
        for direct in (False, True):
            got = []
            for _ in range(2):  # capture, then replay: deterministic
                h_out.zero_()
                step.attend_host(h_tq, tk, tv, h_out, chunks=C, direct_out=direct)
                torch.cuda.synchronize()
                got.append(h_out.clone())
            assert torch.equal(got[0], got[1])
            torch.testing.assert_close(got[0].float(), want.cpu().float(), rtol=2e-2, atol=2e-2)
    # the whole step with in-graph copies (target-Q H2D under capture + select,
    # D2H per unit group): same masks, attention within tolerance, deterministic
    h_dq = dq.cpu().pin_memory()
    got = []
    for _ in range(2):
        h_out.zero_()
        step.step_host(h_dq, dk, h_tq, tk, tv, h_out, chunks=2, direct_out=False)
        torch.cuda.synchronize()
        got.append(h_out.clone())
    assert torch.equal(got[0], got[1])
    torch.testing.assert_close(got[0].float(), want.cpu().float(), rtol=2e-2, atol=2e-2)
    # default with a pinned output: in-graph target-Q H2D, the kernel writes
    # the output directly (one attention launch: bit-exact)
    h_out.zero_()
    step.step_host(h_dq, dk, h_tq, tk, tv, h_out)
    torch.cuda.synchronize()
    assert torch.equal(h_out, want.cpu())


def test_mask_agreement_with_fp64_reference_rows(cuda_ok):
    """masks from the device capture (bf16 inputs, fp32 rows)
    against masks from fp64 reference draft rows on the same inputs."""
    import torch

    from oracle import parity
    from paper_2605_15508_b200 import SparsityConfig
    from paper_2605_15508_b200.verify_step import STSVerifyStep, random_mapping_table, synthetic_inputs

    s = _small_shape()
    step = STSVerifyStep(s, SparsityConfig(budget=0.1), random_mapping_table(s, seed=4), mode="S")
    dq, dk, tq, tk, tv = synthetic_inputs(s, "cuda", seed=9)
    step.step(*step.draft_views(dq, dk), *step.target_views(tq, tk, tv))
    torch.cuda.synchronize()
    agree = parity.mask_agreement(step, dq, dk, list(range(s.target_units)))
    assert agree["recall"] >= 0.99 and agree["min_recall"] >= 0.97, agree


def test_host_api_graph_cache_bounded(cuda_ok):
    """Fresh host buffers on every call: each call captures a graph that holds
    its buffers; the cache stays bounded and every result is right."""
    import torch

    from paper_2605_15508_b200 import SparsityConfig
    from paper_2605_15508_b200.verify_step import STSVerifyStep, random_mapping_table, synthetic_inputs

    s = _small_shape()
    step = STSVerifyStep(s, SparsityConfig(budget=0.1), random_mapping_table(s, seed=2), mode="S")
    dq, dk, tq, tk, tv = synthetic_inputs(s, "cuda", seed=3)
    q, k, v = step.target_views(tq, tk, tv)
    out, _ = step.step(*step.draft_views(dq, dk), q, k, v)
    want = out.cpu()
    for _ in range(step._GRAPH_CACHE + 8):
        h_out = torch.empty(want.shape, dtype=want.dtype).pin_memory()
        step.attend_host(tq.cpu().pin_memory(), tk, tv, h_out)
        torch.cuda.synchronize()
        assert torch.equal(h_out, want)
    assert len(step._graphs) <= step._GRAPH_CACHE
