"""KV offload tier: mask-driven page plans, page copies
from pinned host memory into the HBM pool, and the decode on the pool —
checked against the oracle on the HBM-resident K/V (and bit-identical to the
resident decode)."""

import numpy as np
import pytest

from oracle import sts_oracle as O

pytestmark = pytest.mark.gpu


def _setup(page_sel, context=3000, P=16):
    import torch

    from paper_2605_15508_b200 import SparsityConfig
    from paper_2605_15508_b200.verify_step import STSVerifyStep, VerifyShape, random_mapping_table, synthetic_inputs

    s = VerifyShape(batch=1, context=context, gamma=4, target_layers=3, target_q_heads=8, target_kv_heads=2,
                    head_dim=128, draft_layers=2, draft_q_heads=8, draft_kv_heads=2, draft_head_dim=64)
    step = STSVerifyStep(s, SparsityConfig(budget=0.1, page_size=page_sel), random_mapping_table(s, 3), mode="S")
    dq, dk, tq, tk, tv = synthetic_inputs(s, "cuda", seed=7)
    q, k, v = step.target_views(tq, tk, tv)
    step.capture(*step.draft_views(dq, dk))
    step.build_masks()
    torch.cuda.synchronize()
    return torch, s, step, q, k, v


@pytest.mark.parametrize("page_sel,context", [(16, 3000), (1, 3000), (16, 2048), (8, 1500)])
def test_page_plan_matches_numpy(cuda_ok, page_sel, context):
    from paper_2605_15508_b200.offload import PagedKVOffload

    torch, s, step, q, k, v = _setup(page_sel, context)
    off = PagedKVOffload(step, k.cpu().pin_memory(), v.cpu().pin_memory(), page_size=16)
    off.plan()
    torch.cuda.synchronize()
    idx, cnt = step.idx.cpu().numpy(), step.cnt.cpu().numpy()
    pages, npages, ip = off.pages.cpu().numpy(), off.npages.cpu().numpy(), off.idx_pool.cpu().numpy()
    for u in range(s.target_units):
        lst = idx[u, : cnt[u]]
        pg = lst // 16
        committed = np.unique(pg[pg < off.tail_page0])
        assert npages[u] == committed.size
        assert np.array_equal(pages[u, : npages[u]], committed)
        rank = np.where(pg >= off.tail_page0, off.tail_rank0 + pg - off.tail_page0, np.searchsorted(committed, pg))
        assert np.array_equal(ip[u, : cnt[u]], rank * 16 + lst % 16)
    assert int(step.status.item()) == 0


@pytest.mark.parametrize("page_sel", [16, 1])
def test_offload_strategies_match_resident_and_oracle(cuda_ok, page_sel):
    from paper_2605_15508_b200.offload import PagedKVOffload

    torch, s, step, q, k, v = _setup(page_sel)
    step.attend(q, k, v)
    torch.cuda.synchronize()
    resident = step.out.clone()
    off = PagedKVOffload(step, k.cpu().pin_memory(), v.cpu().pin_memory(), page_size=16, copy_ctas=8)
    for fn in (off.attend_on_demand, off.attend_prefetch):
        step.out.zero_()
        fn(q)
        torch.cuda.synchronize()
        assert torch.equal(step.out, resident), fn.__name__
    assert int(step.status.item()) == 0
    # oracle on the HBM-resident K/V, sampled units
    qf, kf, vf = (x.float().cpu().numpy() for x in (q, k, v))
    idx, cnt = step.idx.cpu().numpy(), step.cnt.cpu().numpy()
    outf = step.out.float().cpu().numpy()
    for u in range(0, s.target_units, 2):
        want, _ = O.block_attention(qf[u], kf[u], vf[u], idx[u, : cnt[u]], causal_base=s.context, rows_per_head=s.rows)
        assert np.abs(outf[u] - want).max() < 2e-2
    if page_sel == 16:  # page-granular masks move only the selected pages
        assert off.bytes_moved() < 0.2 * s.target_units * s.n_kv * s.head_dim * 2 * 2


def test_page_cache_plan_matches_reference_lru(cuda_ok):
    """sts_page_cache_plan over the golden page traces: per step the copied
    pages are exactly the reference simulator's missing pages (specsparse
    offloadsim 'prefetch', tests/golden/offload_lru.json), every used page
    sits in a slot that holds it, and the key lists map to those slots."""
    import json
    from pathlib import Path

    import torch

    from paper_2605_15508_b200._lib import call, ptr

    g = json.loads((Path(__file__).resolve().parent / "golden" / "offload_lru.json").read_text())
    P = 4
    for case in g["cases"]:
        C, NP = case["capacity"], case["n_pages"]
        want = O.lru_prefetch_steps(case["traces"], C)
        assert [len(m) for m in want] == case["missing_per_step"]
        units, ld = 3, C + 1  # three units replay the same trace (per-unit state)
        slot_page = torch.full((units, ld), -1, dtype=torch.int32, device="cuda")
        slot_last = torch.full((units, ld), -1, dtype=torch.int32, device="cuda")
        cp = torch.empty((units, ld), dtype=torch.int32, device="cuda")
        cs = torch.empty((units, ld), dtype=torch.int32, device="cuda")
        nc = torch.empty((units,), dtype=torch.int32, device="cuda")
        status = torch.zeros((1,), dtype=torch.int32, device="cuda")
        for step_no, (pages, miss) in enumerate(zip(case["traces"], want)):
            # each page contributes tokens page*P + {0, P-1} (ascending list)
            toks = np.array(sorted({p * P + o for p in pages for o in (0, P - 1)}), dtype=np.int32)
            idx_ld = max(1, toks.size)
            idx = torch.from_numpy(np.tile(toks, (units, 1)).reshape(units, -1)).cuda() if toks.size else \
                torch.zeros((units, 1), dtype=torch.int32, device="cuda")
            cnt = torch.full((units,), toks.size, dtype=torch.int32, device="cuda")
            ip = torch.empty_like(idx)
            call("sts_page_cache_plan", ptr(idx), idx_ld, ptr(cnt), units, P, NP, C, ptr(slot_page), ptr(slot_last),
                 ld, C, step_no, ptr(cp), ptr(cs), ptr(nc), ptr(ip), ptr(status), None)
            torch.cuda.synchronize()
            assert int(status.item()) == 0
            sp, ncn, cpn, csn, ipn = (x.cpu().numpy() for x in (slot_page, nc, cp, cs, ip))
            for u in range(units):
                assert ncn[u] == len(miss), (step_no, u)
                assert list(cpn[u, : ncn[u]]) == sorted(miss)
                assert all(sp[u, csn[u, i]] == cpn[u, i] for i in range(ncn[u]))
                slot = ipn[u, : toks.size] // P
                assert np.array_equal(sp[u, slot], toks // P)  # every key's slot holds its page
                assert np.array_equal(ipn[u, : toks.size] % P, toks % P)


def test_resident_pool_across_steps_matches_hbm(cuda_ok):
    """The resident pool over three verify steps whose masks drift: each step
    copies only its missing pages and the decode on the pool equals the
    HBM-resident decode bit for bit."""
    from paper_2605_15508_b200.offload import PagedKVOffload

    torch, s, step, q, k, v = _setup(16)
    off = PagedKVOffload(step, k.cpu().pin_memory(), v.cpu().pin_memory(), page_size=16, copy_ctas=8, resident=True)
    g = torch.Generator(device="cuda").manual_seed(11)
    moved = []
    for it in range(3):
        if it:
            step.draft_rows.mul_(1 + 0.3 * torch.rand(step.draft_rows.shape, generator=g, device="cuda"))
            step.build_masks()
        step.attend(q, k, v)
        torch.cuda.synchronize()
        resident = step.out.clone()
        step.out.zero_()
        off.attend_prefetch(q)
        torch.cuda.synchronize()
        assert torch.equal(step.out, resident), it
        moved.append(off.bytes_moved())
    assert int(step.status.item()) == 0
    assert moved[1] < moved[0] and moved[2] < moved[0]  # later steps copy only what changed


def test_page_cache_capacity_flag(cuda_ok):
    """A step needing more committed pages than the pool's slots sets
    STS_DEV_IDX_CAPACITY (the reference raises ConfigError for the same trace,
    src/offloadsim.py:122-126)."""
    import torch

    from paper_2605_15508_b200._lib import call, ptr

    P, C, NP = 4, 3, 32
    toks = torch.tensor([[p * P for p in (1, 5, 9, 13, 17)]], dtype=torch.int32, device="cuda")
    cnt = torch.tensor([5], dtype=torch.int32, device="cuda")
    sp = torch.full((1, C + 1), -1, dtype=torch.int32, device="cuda")
    sl = torch.full((1, C + 1), -1, dtype=torch.int32, device="cuda")
    cp, cs = torch.empty_like(sp), torch.empty_like(sp)
    nc = torch.empty((1,), dtype=torch.int32, device="cuda")
    ip = torch.empty_like(toks)
    status = torch.zeros((1,), dtype=torch.int32, device="cuda")
    call("sts_page_cache_plan", ptr(toks), 5, ptr(cnt), 1, P, NP, C, ptr(sp), ptr(sl), C + 1, C, 0, ptr(cp), ptr(cs),
         ptr(nc), ptr(ip), ptr(status), None)
    torch.cuda.synchronize()
    assert int(status.item()) & 0x1
    assert int(nc.item()) == C
