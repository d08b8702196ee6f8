"""Block-sparse prefill on tcgen05: tile-granular masks
(128-row query tiles, 64-key blocks chosen per (kv-head, tile) by the GPU
select + the causal diagonal) vs the fp64 oracle on the bf16-rounded inputs
(2e-2), dense mode vs causal attention, block lists vs a numpy restatement
of the selection."""

import numpy as np
import pytest

from oracle import sts_oracle as O

pytestmark = pytest.mark.gpu
TILE, BLK = 128, 64


def _inputs(n, hq, hkv, d, seed=0):
    import torch

    g = torch.Generator(device="cuda").manual_seed(seed)
    q = torch.randn((hq, n, d), generator=g, device="cuda").bfloat16()
    k = torch.randn((hkv, n, d), generator=g, device="cuda").bfloat16()
    v = torch.randn((hkv, n, d), generator=g, device="cuda").bfloat16()
    tiles = -(-n // TILE)
    width = -(-n // 4) * 4
    scores = torch.softmax(2 * torch.randn((hkv * tiles, width), generator=g, device="cuda"), -1).contiguous()
    return q, k, v, scores


def _oracle_tile(qf, kf, vf, keys, T, n):
    rows = slice(T * TILE, min(T * TILE + TILE, n))
    out, _ = O.block_attention(qf[rows], kf, vf, np.asarray(keys), causal_base=T * TILE, rows_per_head=TILE)
    return out


@pytest.mark.parametrize("n,hq,hkv,d", [(1000, 4, 2, 128), (512, 2, 1, 64), (1280, 4, 1, 128)])
def test_blocksparse_prefill_vs_oracle(cuda_ok, n, hq, hkv, d):
    import torch

    from paper_2605_15508_b200 import kernels

    q, k, v, scores = _inputs(n, hq, hkv, d)
    idx, cnt = kernels.prefill_tile_select(scores, budget=0.1, n=n)
    status = torch.zeros((1,), dtype=torch.int32, device="cuda")
    out = kernels.prefill_blocksparse(q, k, v, idx=idx, cnt=cnt, status=status)
    dense = kernels.prefill_blocksparse(q, k, v, status=status)
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    qf, kf, vf = (x.float().cpu().numpy() for x in (q, k, v))
    of, df = out.float().cpu().numpy(), dense.float().cpu().numpy()
    ih, ch, sc = idx.cpu().numpy(), cnt.cpu().numpy(), scores.cpu().numpy()
    tiles = -(-n // TILE)
    ocfg = O.OracleSparsityConfig(0.1, BLK, False, False, 0)
    for h in range(hq):
        kv = h // (hq // hkv)
        for T in range(tiles):
            r = kv * tiles + T
            committed = ih[r, : ch[r]]
            if T > 0:  # the block selection is the reference page rule over the committed context
                assert np.array_equal(committed, O.select_row(sc[r, : T * TILE], ocfg))
                assert ch[r] % BLK == 0
            else:
                assert ch[r] == 0
            keys = np.union1d(committed, np.arange(T * TILE, min(T * TILE + TILE, n)))
            rows = slice(T * TILE, min(T * TILE + TILE, n))
            want = _oracle_tile(qf[h], kf[kv], vf[kv], keys, T, n)
            assert np.abs(of[h, rows] - want).max() < 2e-2, (h, T)
            want_dense = _oracle_tile(qf[h], kf[kv], vf[kv], np.arange(min(T * TILE + TILE, n)), T, n)
            assert np.abs(df[h, rows] - want_dense).max() < 2e-2, (h, T, "dense")


@pytest.mark.parametrize("n,hq,hkv,d", [(6000, 8, 2, 128), (5000, 16, 4, 64)])
def test_blocksparse_prefill_persistent_many_items(cuda_ok, n, hq, hkv, d):
    """More work items (tiles x q-heads) than SMs, so every persistent CTA runs
    several items back to back (double-buffered Q, barrier phases carried
    across items, O drained between items): dense and block-sparse outputs vs
    a PyTorch fp32 reference of the same masks (bf16 tolerance), plus a few
    tiles against the fp64 oracle."""
    import torch

    from paper_2605_15508_b200 import kernels

    q, k, v, scores = _inputs(n, hq, hkv, d, seed=3)
    tiles = -(-n // TILE)
    assert tiles * hq > torch.cuda.get_device_properties(0).multi_processor_count
    idx, cnt = kernels.prefill_tile_select(scores, budget=0.1, n=n)
    status = torch.zeros((1,), dtype=torch.int32, device="cuda")
    out = kernels.prefill_blocksparse(q, k, v, idx=idx, cnt=cnt, status=status)
    dense = kernels.prefill_blocksparse(q, k, v, status=status)
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    g = hq // hkv
    qf, kf, vf = q.float(), k.float().repeat_interleave(g, 0), v.float().repeat_interleave(g, 0)
    pos = torch.arange(n, device="cuda")
    causal = pos[None, :] <= pos[:, None]
    ref_dense = torch.nn.functional.scaled_dot_product_attention(qf, kf, vf, attn_mask=causal)
    assert (dense.float() - ref_dense).abs().max().item() < 2e-2
    # per (kv-head, tile): selected committed keys + the tile's causal diagonal
    allowed = torch.zeros((hkv, n, n), dtype=torch.bool, device="cuda")
    ih, ch = idx.cpu().numpy(), cnt.cpu().numpy()
    for kv in range(hkv):
        for T in range(tiles):
            r0, r1 = T * TILE, min(T * TILE + TILE, n)
            sel = torch.from_numpy(ih[kv * tiles + T, : ch[kv * tiles + T]].astype(np.int64)).cuda()
            allowed[kv, r0:r1, sel] = True
            allowed[kv, r0:r1, r0:r1] = causal[r0:r1, r0:r1]
    ref = torch.nn.functional.scaled_dot_product_attention(qf, kf, vf, attn_mask=allowed.repeat_interleave(g, 0))
    assert (out.float() - ref).abs().max().item() < 2e-2
    # a few tiles against the fp64 oracle
    qn, kn, vn = (x.float().cpu().numpy() for x in (q, k, v))
    of = out.float().cpu().numpy()
    for h, T in ((0, tiles - 1), (hq - 1, tiles // 2), (hq // 2, 1)):
        kv = h // g
        committed = ih[kv * tiles + T, : ch[kv * tiles + T]]
        keys = np.union1d(committed, np.arange(T * TILE, min(T * TILE + TILE, n)))
        rows = slice(T * TILE, min(T * TILE + TILE, n))
        assert np.abs(of[h, rows] - _oracle_tile(qn[h], kn[kv], vn[kv], keys, T, n)).max() < 2e-2, (h, T)
