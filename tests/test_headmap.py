"""Algorithm 1 (offline head mapping): the oracle against the
reference's own find_head_mapping outputs (tests/golden/headmap.npz, recorded
by make_golden.py from /root/reference), and the GPU implementation against
the same golden vectors (bit-exact: integer overlap counts)."""

import json
from types import SimpleNamespace

import numpy as np
import pytest

from conftest import load_golden
from oracle import sts_oracle as O

DRAFT = [(l, h) for l in range(2) for h in range(3)]
TARGET = [(l, h) for l in range(2) for h in range(4)]


def _golden():
    g = load_golden("headmap.npz")
    samples = []
    for si, n in enumerate(g["lengths"]):
        draft = {dh: g[f"s{si}_d{dh[0]}_{dh[1]}"] for dh in DRAFT}
        target = {th: g[f"s{si}_t{th[0]}_{th[1]}"] for th in TARGET}
        samples.append((int(n), draft, target))
    return samples, json.loads(str(g["result"]))


def test_oracle_matches_reference_algorithm1():
    samples, result = _golden()
    for k, rows in result.items():
        got = O.find_head_mapping([(d, t) for _, d, t in samples], DRAFT, TARGET, int(k))
        for tl, th, dl, dh, score in rows:
            assert got[(tl, th)] == ((dl, dh), score), (k, tl, th)


@pytest.mark.gpu
def test_gpu_algorithm1_matches_reference(cuda_ok):
    from paper_2605_15508_b200 import find_head_mapping

    samples, result = _golden()
    ts = SimpleNamespace(
        samples=[SimpleNamespace(length=n, draft=d, target=t) for n, d, t in samples],
        draft_config=SimpleNamespace(layers=2, heads=3), target_config=SimpleNamespace(layers=2, heads=4))
    for k, rows in result.items():
        mp = find_head_mapping(ts, int(k))
        for tl, th, dl, dh, score in rows:
            assert mp.entries[(tl, th)] == ((dl, dh), score), (k, tl, th)


@pytest.mark.gpu
@pytest.mark.parametrize("Ta,Tb,W", [(1, 1, 4), (70, 33, 100), (64, 130, 4096), (5, 200, 36), (3, 2, 100000), (300, 129, 1028)])
def test_gpu_bitset_overlap_matches_popcount(cuda_ok, Ta, Tb, W):
    """sts_bitset_overlap (tiled AND + popcount) = numpy's popcount of the ANDs,
    accumulated into the existing scores (ragged tiles and chunks)."""
    import torch

    from paper_2605_15508_b200 import _lib
    from paper_2605_15508_b200._lib import call, ptr, stream_handle

    _lib.load()
    rng = np.random.default_rng(Ta * 1000 + Tb + W)
    a = rng.integers(0, 2**32, size=(Ta, W), dtype=np.uint64).astype(np.uint32)
    b = rng.integers(0, 2**32, size=(Tb, W), dtype=np.uint64).astype(np.uint32)
    a[0, :] = 0xFFFFFFFF  # saturated row
    init = rng.integers(0, 1000, size=(Ta, Tb)).astype(np.int64)
    da = torch.from_numpy(a.view(np.int32)).cuda()
    db = torch.from_numpy(b.view(np.int32)).cuda()
    scores = torch.from_numpy(init.copy()).cuda()
    call("sts_bitset_overlap", ptr(da), Ta, ptr(db), Tb, W, ptr(scores), stream_handle())
    torch.cuda.synchronize()
    pc = np.unpackbits((a[:, None, :] & b[None, :, :]).view(np.uint8), axis=-1).sum(axis=-1)
    np.testing.assert_array_equal(scores.cpu().numpy(), init + pc)
