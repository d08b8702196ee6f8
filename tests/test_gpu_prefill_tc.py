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
