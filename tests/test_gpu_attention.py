"""GPU parity of the gathered sparse flash-decode and the LSE merge.

fp32 path: rtol 1e-5 / atol 1e-6 vs the fp64 reference math
(src/sparsity.py:152-173; tolerance of pkg/tests/test_acceptance.py:63).
bf16 path: rtol/atol 2e-2 vs the fp64 oracle evaluated on the same
bf16-rounded inputs (north-star bf16 tolerance).
"""

import math

import numpy as np
import pytest

from conftest import load_golden, unpack
from oracle import sts_oracle as O

pytestmark = pytest.mark.gpu

RTOL32, ATOL32 = 1e-5, 1e-6
TOL16 = 2e-2


def test_golden_sparse_attention(cuda_ok):
    from paper_2605_15508_b200 import sparse_attention

    g = load_golden("sparse_attention.npz")
    qo = ko = oo = 0
    masks = unpack(g["mask"], g["mask_offs"])
    for (n, d), mask in zip(g["shapes"], masks):
        q = g["q"][qo : qo + d]; qo += d
        k = g["k"][ko : ko + n * d].reshape(n, d)
        v = g["v"][ko : ko + n * d].reshape(n, d); ko += n * d
        want = g["out"][oo : oo + d]; oo += d
        np.testing.assert_allclose(sparse_attention(q, k, v, mask), want, rtol=RTOL32, atol=ATOL32)


def test_reference_known_answers_and_errors(cuda_ok):
    from paper_2605_15508_b200 import ContractViolation, sparse_attention

    rng = np.random.default_rng(3)
    q, k, v = rng.standard_normal(6), rng.standard_normal((10, 6)), rng.standard_normal((10, 6))
    np.testing.assert_allclose(sparse_attention(q, k, v, np.array([4])), v[4], rtol=1e-6)  # mask {4} -> v[4]
    np.testing.assert_allclose(sparse_attention(q, k, v, np.arange(10)),
                               O.sparse_attention(q, k, v, np.arange(10)), rtol=RTOL32, atol=ATOL32)
    with pytest.raises(ContractViolation):
        sparse_attention(q, k, v, np.array([], dtype=np.int64))
    with pytest.raises(ContractViolation):
        sparse_attention(q, k, v, np.array([10]))


def _case(rng, U, M, N, d, R, base, cnt_range, dtype):
    import torch

    q = rng.standard_normal((U, M, d)).astype(np.float32)
    k = rng.standard_normal((U, N, d)).astype(np.float32)
    v = rng.standard_normal((U, N, d)).astype(np.float32)
    if dtype == "bf16":
        q, k, v = (torch.from_numpy(x).bfloat16().float().numpy() for x in (q, k, v))
    lists = []
    for u in range(U):
        c = int(rng.integers(*cnt_range))
        sel = np.sort(rng.choice(base, size=min(c, base), replace=False))
        lists.append(np.concatenate([sel, np.arange(base, base + R)]))
    ld = max(len(x) for x in lists) + 3
    idx = np.zeros((U, ld), np.int32)
    cnt = np.zeros(U, np.int32)
    for u, x in enumerate(lists):
        idx[u, : len(x)] = x
        cnt[u] = len(x)
    return q, k, v, lists, idx, cnt


def _to_dev(x, dtype):
    import torch

    t = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    return t.bfloat16() if dtype == "bf16" and t.dtype == torch.float32 else t


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("d,G,R", [(64, 1, 5), (128, 4, 5), (64, 4, 5), (128, 7, 5), (128, 8, 5), (128, 1, 1)])
@pytest.mark.parametrize("splits", [1, 3])
def test_stacked_rows_causal_tail(cuda_ok, dtype, d, G, R, splits):
    """Mode-S layout: M = G*R rows share one key list; in-block keys obey the
    per-row causal rule pos - base <= r % R."""
    from paper_2605_15508_b200 import kernels

    rng = np.random.default_rng(d * 100 + G * 10 + R + splits)
    U, base = 6, 700
    M, N = G * R, base + R
    q, k, v, lists, idx, cnt = _case(rng, U, M, N, d, R, base, (1, 400), dtype)
    out, lse = kernels.sparse_decode(_to_dev(q, dtype), _to_dev(k, dtype), _to_dev(v, dtype), idx=_to_dev(idx, dtype),
                                     cnt=_to_dev(cnt, dtype), causal_base=base, rows_per_head=R, splits=splits)
    out = out.float().cpu().numpy()
    lse = lse.cpu().numpy()
    for u in range(U):
        want, wlse = O.block_attention(q[u], k[u], v[u], lists[u], causal_base=base, rows_per_head=R)
        if dtype == "f32":
            np.testing.assert_allclose(out[u], want, rtol=RTOL32, atol=ATOL32)
            np.testing.assert_allclose(lse[u], wlse, rtol=1e-5, atol=1e-5)
        else:
            np.testing.assert_allclose(out[u], want, rtol=TOL16, atol=TOL16)
            np.testing.assert_allclose(lse[u], wlse, rtol=1e-3, atol=1e-2)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_member_bits_mode_r(cuda_ok, dtype):
    """Mode R: per-(row, key) membership bits select each row's own mask."""
    from paper_2605_15508_b200 import kernels

    rng = np.random.default_rng(11)
    U, G, R, d, N = 4, 4, 5, 128, 1200
    M = G * R
    q = rng.standard_normal((U, M, d)).astype(np.float32)
    k = rng.standard_normal((U, N, d)).astype(np.float32)
    v = rng.standard_normal((U, N, d)).astype(np.float32)
    if dtype == "bf16":
        import torch
        q, k, v = (torch.from_numpy(x).bfloat16().float().numpy() for x in (q, k, v))
    ld = N
    idx = np.zeros((U, ld), np.int32)
    mem = np.zeros((U, ld), np.uint32)
    cnt = np.zeros(U, np.int32)
    row_masks = []
    for u in range(U):
        masks = [np.sort(rng.choice(N, size=int(rng.integers(1, 300)), replace=False)) for _ in range(M)]
        union = np.unique(np.concatenate(masks))
        bits = np.zeros(union.size, np.uint32)
        for r, m in enumerate(masks):
            bits[np.searchsorted(union, m)] |= np.uint32(1 << r)
        idx[u, : union.size] = union
        mem[u, : union.size] = bits
        cnt[u] = union.size
        row_masks.append(masks)
    out, _ = kernels.sparse_decode(_to_dev(q, dtype), _to_dev(k, dtype), _to_dev(v, dtype), idx=_to_dev(idx, dtype),
                                   cnt=_to_dev(cnt, dtype), member=_to_dev(mem.view(np.int32), dtype), splits=2)
    out = out.float().cpu().numpy()
    tol = (RTOL32, ATOL32) if dtype == "f32" else (TOL16, TOL16)
    for u in range(U):
        for r in range(M):
            want = O.sparse_attention(q[u, r], k[u], v[u], row_masks[u][r])
            np.testing.assert_allclose(out[u, r], want, rtol=tol[0], atol=tol[1])


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_dense_path_equals_full_mask(cuda_ok, dtype):
    """idx=None (dense baseline) == the same rows with an explicit full list."""
    from paper_2605_15508_b200 import kernels

    rng = np.random.default_rng(5)
    U, G, R, d, base = 3, 4, 5, 128, 2000
    N = base + R
    q, k, v, _, _, _ = _case(rng, U, G * R, N, d, R, base, (1, 2), dtype)
    out, lse = kernels.sparse_decode(_to_dev(q, dtype), _to_dev(k, dtype), _to_dev(v, dtype), n_dense=N,
                                     causal_base=base, rows_per_head=R)
    out = out.float().cpu().numpy()
    for u in range(U):
        want, _ = O.block_attention(q[u], k[u], v[u], np.arange(N), causal_base=base, rows_per_head=R)
        tol = (RTOL32, ATOL32) if dtype == "f32" else (TOL16, TOL16)
        np.testing.assert_allclose(out[u], want, rtol=tol[0], atol=tol[1])


def test_lse_merge_of_shards_equals_union(cuda_ok):
    """Sequence-shard partials merged by sts_lse_merge == attention over the union."""
    import torch

    from paper_2605_15508_b200 import kernels

    rng = np.random.default_rng(9)
    U, G, R, d, base, P = 4, 4, 5, 128, 4000, 4
    M, N = G * R, base + R
    q, k, v, lists, _, _ = _case(rng, U, M, N, d, R, base, (100, 900), "f32")
    bounds = O.shard_bounds(N, P, align=16)
    o_parts, l_parts = [], []
    for lo, hi in bounds:
        loc = [x[(x >= lo) & (x < hi)] - lo for x in lists]
        ld = max(1, max(len(x) for x in loc))
        idx = np.zeros((U, ld), np.int32)
        cnt = np.array([len(x) for x in loc], np.int32)
        for u, x in enumerate(loc):
            idx[u, : len(x)] = x
        o, l = kernels.sparse_decode(_to_dev(q, "f32"), _to_dev(k[:, lo:hi], "f32").contiguous(),
                                     _to_dev(v[:, lo:hi], "f32").contiguous(), idx=_to_dev(idx, "f32"),
                                     cnt=_to_dev(cnt, "f32"), causal_base=base, rows_per_head=R, pos_offset=lo)
        o_parts.append(o.reshape(U * M, d))
        l_parts.append(l.reshape(U * M))
    merged, lse = kernels.lse_merge(torch.stack(o_parts), torch.stack(l_parts))
    merged = merged.cpu().numpy().reshape(U, M, d)
    for u in range(U):
        want, wl = O.block_attention(q[u], k[u], v[u], lists[u], causal_base=base, rows_per_head=R)
        np.testing.assert_allclose(merged[u], want, rtol=RTOL32, atol=ATOL32)
        np.testing.assert_allclose(lse.cpu().numpy().reshape(U, M)[u], wl, rtol=1e-5, atol=1e-5)


def test_row_union(cuda_ok):
    import torch

    from paper_2605_15508_b200 import kernels

    rng = np.random.default_rng(13)
    L, ld, n = 30, 300, 1000
    lists = [np.sort(rng.choice(n, size=int(rng.integers(1, ld)), replace=False)) for _ in range(L)]
    idx = np.zeros((L, ld), np.int32)
    cnt = np.array([len(x) for x in lists], np.int32)
    for i, x in enumerate(lists):
        idx[i, : len(x)] = x
    src = rng.integers(0, L, size=(5, 20)).astype(np.int32)
    u_idx, mem, u_cnt = kernels.row_union(torch.from_numpy(idx).cuda(), torch.from_numpy(cnt).cuda(),
                                          torch.from_numpy(src).cuda(), M=20, n_max=n)
    u_idx, mem, u_cnt = u_idx.cpu().numpy(), mem.cpu().numpy().view(np.uint32), u_cnt.cpu().numpy()
    for u in range(5):
        want = np.unique(np.concatenate([lists[s] for s in src[u]]))
        np.testing.assert_array_equal(u_idx[u, : u_cnt[u]], want)
        for r in range(20):
            have = u_idx[u, : u_cnt[u]][(mem[u, : u_cnt[u]] >> r) & 1 == 1]
            np.testing.assert_array_equal(have, lists[src[u, r]])


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_interleaved_kv_row_stride(cuda_ok, dtype):
    """K|V interleaved per token ([U, N, 2, d]) through the row-stride views."""
    import torch

    from paper_2605_15508_b200 import kernels

    rng = np.random.default_rng(21)
    U, G, R, d, base = 3, 4, 5, 128, 900
    M, N = G * R, base + R
    q, k, v, lists, idx, cnt = _case(rng, U, M, N, d, R, base, (10, 300), dtype)
    kv = np.stack([k, v], axis=2)  # [U, N, 2, d]
    kvd = _to_dev(kv, dtype)
    out, _ = kernels.sparse_decode(_to_dev(q, dtype), kvd[:, :, 0, :], kvd[:, :, 1, :], idx=_to_dev(idx, dtype),
                                   cnt=_to_dev(cnt, dtype), causal_base=base, rows_per_head=R, splits=2)
    out = out.float().cpu().numpy()
    tol = (RTOL32, ATOL32) if dtype == "f32" else (TOL16, TOL16)
    for u in range(U):
        want, _ = O.block_attention(q[u], k[u], v[u], lists[u], causal_base=base, rows_per_head=R)
        np.testing.assert_allclose(out[u], want, rtol=tol[0], atol=tol[1])


def test_stream_k_schedule_variant(cuda_ok):
    """The attention parity suite again with the cluster schedule disabled
    (STS_VERIFY_CLUSTER=0: every launch takes the stream-K + piece-merge path),
    in a subprocess because the library reads the knob once."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    env = dict(os.environ, STS_VERIFY_CLUSTER="0")
    r = subprocess.run([sys.executable, "-m", "pytest", str(root / "tests" / "test_gpu_attention.py"), "-q", "-x",
                        "-p", "no:cacheprovider", "-k", "not stream_k_schedule_variant"],
                       env=env, cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_host_resident_kv_offload(cuda_ok):
    """KV offload tier: the caches in pinned host memory, read by the same
    kernel over the host link (only the selected rows cross it) — results
    identical to the HBM-resident run."""
    import torch

    from paper_2605_15508_b200 import kernels

    rng = np.random.default_rng(9)
    U, M, d, N = 6, 20, 128, 2000
    q = torch.from_numpy(rng.standard_normal((U, M, d)).astype(np.float32)).bfloat16().cuda()
    k = torch.from_numpy(rng.standard_normal((U, N, d)).astype(np.float32)).bfloat16()
    v = torch.from_numpy(rng.standard_normal((U, N, d)).astype(np.float32)).bfloat16()
    sel = np.stack([np.sort(rng.choice(N, 300, replace=False)) for _ in range(U)]).astype(np.int32)
    idx = torch.from_numpy(sel).cuda()
    cnt = torch.full((U,), 300, dtype=torch.int32, device="cuda")
    dev_out, dev_lse = kernels.sparse_decode(q, k.cuda(), v.cuda(), idx=idx, cnt=cnt)
    kh, vh = k.pin_memory(), v.pin_memory()
    host_out, host_lse = kernels.sparse_decode(q, kh, vh, idx=idx, cnt=cnt, host_kv=True)
    torch.cuda.synchronize()
    assert torch.equal(dev_out, host_out) and torch.equal(dev_lse, host_lse)
    with pytest.raises(ValueError):
        kernels.sparse_decode(q, k, v, idx=idx, cnt=cnt)  # pageable host memory is refused
