"""GPU parity of sparse prefill attention (STS-PD): every
query row attends its own mask — masks from the GPU draft_masks_prefill
(bit-exact vs the reference golden, tests/test_gpu_select.py), attention vs the
oracle's sparse_attention per row (fp32: rtol 1e-5; bf16: 2e-2)."""

import numpy as np
import pytest

from oracle import sts_oracle as O

pytestmark = pytest.mark.gpu


def _prefill_rows(rng, n):
    mat = np.zeros((n, n), dtype=np.float32)
    for t in range(n):
        z = 2.0 * rng.standard_normal(t + 1)
        w = np.exp(z - z.max())
        mat[t, : t + 1] = w / w.sum()
    return mat


def test_reference_named_prefill_matches_oracle(cuda_ok):
    from paper_2605_15508_b200 import SparsityConfig, draft_masks_prefill, sparse_prefill_attention

    rng = np.random.default_rng(0)
    n, d = 300, 64
    mat = _prefill_rows(rng, n)
    cfg = SparsityConfig(budget=0.1, include_sink=True, recent_window=4)
    masks = draft_masks_prefill({(0, 0): mat}, cfg)[(0, 0)]
    ocfg = O.OracleSparsityConfig(0.1, 1, True, True, 4)
    for t in (0, 1, 17, 299):
        np.testing.assert_array_equal(masks[t], O.select_row(mat[t, : t + 1], ocfg))
    q = rng.standard_normal((n, d)).astype(np.float32)
    k = rng.standard_normal((n, d)).astype(np.float32)
    v = rng.standard_normal((n, d)).astype(np.float32)
    got = sparse_prefill_attention(q, k, v, masks)
    want = np.stack([O.sparse_attention(q[t], k, v, masks[t]) for t in range(n)])
    np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-6)


def test_reference_named_prefill_contract_errors(cuda_ok):
    from paper_2605_15508_b200 import ContractViolation, sparse_prefill_attention

    q = np.zeros((3, 8), np.float32)
    k = np.zeros((3, 8), np.float32)
    with pytest.raises(ContractViolation, match="empty"):
        sparse_prefill_attention(q, k, k, [np.array([0]), np.array([], np.int64), np.array([2])])
    with pytest.raises(ContractViolation, match="causal"):
        sparse_prefill_attention(q, k, k, [np.array([0]), np.array([2]), np.array([2])])


@pytest.mark.parametrize("G,M,d", [(2, 4, 128), (3, 1, 64)])
def test_batched_bf16_prefill_gqa(cuda_ok, G, M, d):
    """Batched device path: G K/V blocks x n rows x M heads sharing a row mask
    (mode-S style GQA prefill), masks from the GPU selection of the summed rows."""
    import torch

    from paper_2605_15508_b200 import kernels

    rng = np.random.default_rng(G * 10 + M)
    n = 257
    rows = np.concatenate([_prefill_rows(rng, n) for _ in range(G)])  # [G*n, n]
    scores = torch.from_numpy(rows).cuda()
    row_len = torch.from_numpy(np.tile(np.arange(1, n + 1, dtype=np.int32), G)).cuda()
    idx, cnt = kernels.select_topk(scores, row_len=row_len, budget=0.125, include_current=True)
    q = torch.from_numpy(rng.standard_normal((G, n, M, d)).astype(np.float32)).bfloat16().cuda()
    k = torch.from_numpy(rng.standard_normal((G, n, d)).astype(np.float32)).bfloat16().cuda()
    v = torch.from_numpy(rng.standard_normal((G, n, d)).astype(np.float32)).bfloat16().cuda()
    out, lse = kernels.sparse_prefill(q, k, v, idx=idx, cnt=cnt)
    torch.cuda.synchronize()
    qf, kf, vf = q.float().cpu().numpy(), k.float().cpu().numpy(), v.float().cpu().numpy()
    of = out.float().cpu().numpy()
    ic, cc = idx.cpu().numpy(), cnt.cpu().numpy()
    for g in range(G):
        for t in (0, 1, 5, 128, n - 1):
            r = g * n + t
            sel = ic[r, : cc[r]]
            assert sel.max() <= t
            want, _ = O.block_attention(qf[g, t], kf[g], vf[g], sel)
            np.testing.assert_allclose(of[g, t], want, rtol=2e-2, atol=2e-2)
