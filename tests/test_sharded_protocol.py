"""CPU (gloo, world_size 2 and 3) checks of the sequence-sharded protocol.

The collective plumbing of paper_2605_15508_b200.sharded (``run``: the
torch.distributed servicing of a rank's protocol) is exercised with real
multi-process gloo groups, driving the oracle's restatement of the
radix-round protocol (oracle.dist_select_protocol — the same collective
sequence as DistSelector).  The union of the ranks' selections must equal
topk_indices of the concatenated row (src/numkit.py:74-86) bit for bit.
The kernels themselves are covered on the GPU by tests/test_gpu_sharded.py.
"""

import os
import socket

import numpy as np
import pytest

from oracle import sts_oracle as O


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, rows_np, n, k, q):
    import torch.distributed as dist

    from paper_2605_15508_b200 import sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = sharded.shard_bounds(n, world)[rank]
        proto = O.dist_select_protocol(rows_np[:, lo:hi], lo, n, k, rank, world)
        out = sharded.run(proto)
        q.put((rank, [o.tolist() for o in out]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_sharded_topk_equals_global(world):
    import torch.multiprocessing as mp

    rng = np.random.default_rng(world)
    n, rows = 700, 4
    x = (np.round(rng.random((rows, n)) * 32) / 32).astype(np.float32)  # tie-heavy
    x[1] = np.float32(0.5)  # a row of all ties
    k = 123
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, x, n, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(rows):
        union = np.sort(np.concatenate([np.asarray(got[w][r], dtype=np.int64) for w in range(world)]))
        np.testing.assert_array_equal(union, O.topk_indices(x[r], k))


def test_oracle_protocol_lockstep_matches_topk():
    """The same protocol driven in-process (sharded.run_lockstep) for many
    shard counts, budgets and the dense fallback."""
    from paper_2605_15508_b200 import sharded

    rng = np.random.default_rng(5)
    for trial in range(12):
        n = int(rng.integers(20, 900))
        x = (np.round(rng.random((3, n)) * 16) / 16).astype(np.float32)
        P = int(rng.integers(1, 6))
        k = int(rng.integers(1, n + 3))
        bounds = sharded.shard_bounds(n, P)
        outs = sharded.run_lockstep([O.dist_select_protocol(x[:, lo:hi], lo, n, k, r, P)
                                     for r, (lo, hi) in enumerate(bounds)])
        for row in range(3):
            union = np.sort(np.concatenate([o[row] for o in outs]))
            want = O.topk_indices(x[row], k) if k < n else np.arange(n)
            np.testing.assert_array_equal(union, want)


def test_shard_bounds_page_aligned():
    from paper_2605_15508_b200 import sharded

    for n, P, a in [(1048581, 8, 16), (32773, 3, 1), (100, 8, 16), (5, 2, 1)]:
        b = sharded.shard_bounds(n, P, a)
        assert b[0][0] == 0 and b[-1][1] == n
        assert all(lo % a == 0 for lo, hi in b if hi > lo)
        assert all(b[i][1] == b[i + 1][0] for i in range(P - 1))
        assert b == O.shard_bounds(n, P, a)
