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
