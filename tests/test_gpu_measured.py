"""Parity at the configurations the bench measures (VERDICT r1 "next" #1).

The headline numbers come from kernel instances the small-shape tests never
reach: at c2 (256 units x 3,282 keys) the attention runs as 3-CTA clusters,
at c3 (M = 35, 128K x batch 8) as stream-K with the chunk-parallel long-row
select, at c4 (1M context) through the sharded path at P = 1.  These tests run
exactly those shapes, with the same schedule resolution the bench uses, and
check a seeded sample of units (every layer represented) against the CPU
oracle: masks bit-exact (``oracle.parity`` -> ``mode_s_index_list`` on the
GPU's own draft rows), attention within the bf16 tolerance 2e-2 (fp64
``block_attention_rows``).  Reference math: src/sparsity.py:86-112, :152-173;
src/specdec.py:219-233.

Each big configuration frees its buffers before the next one (c4 holds
~155 GB of caches on one 180 GB B200).
"""

import gc

import numpy as np
import pytest

from oracle import parity

pytestmark = pytest.mark.gpu


@pytest.fixture
def free_gpu():
    import torch

    yield
    gc.collect()
    torch.cuda.empty_cache()


def _run_step(name, schedule=0, page_size=1, sample=32, **overrides):
    import torch

    from paper_2605_15508_b200 import SparsityConfig, _lib
    from paper_2605_15508_b200.verify_step import STSVerifyStep, config_shape, random_mapping_table, synthetic_inputs

    s = config_shape(name, **overrides)
    cfg = SparsityConfig(budget=0.1, page_size=page_size)
    step = STSVerifyStep(s, cfg, random_mapping_table(s, seed=5), mode="S", schedule=schedule)
    dq, dk, tq, tk, tv = synthetic_inputs(s, "cuda", seed=0)
    q, k, v = step.target_views(tq, tk, tv)
    out, _ = step.step(*step.draft_views(dq, dk), q, k, v)
    torch.cuda.synchronize()
    assert step.status.item() == 0, f"device status {step.status.item()}"
    units = parity.sample_units(s.batch, s.target_layers, s.target_kv_heads, sample, seed=1)
    res = parity.check_units(step, q, k, v, out, units)
    plan = _lib.load().sts_sparse_decode_schedule(s.target_units, step.M, s.head_dim, step.idx_ld, schedule)
    return step, res, plan


def _assert_ok(res):
    assert res["masks_bit_exact"], f"mask mismatch in units {res['mask_mismatch_units']}"
    assert res["attention_ok"], f"attention error {res['max_abs_err']} > {res['tol']}"


def test_c2_headline_instance(cuda_ok, free_gpu):
    """The exact c2 workload of the headline (auto schedule: 3-CTA clusters)."""
    step, res, plan = _run_step("c2")
    assert plan == 3, f"c2 auto schedule resolved to {plan}, the bench instance is 3-CTA clusters"
    assert step._dist is None  # 32K rows: the single-CTA select
    _assert_ok(res)


@pytest.mark.parametrize("schedule", [1, 2, 4, 6, 8])
def test_c2_forced_schedules(cuda_ok, free_gpu, schedule):
    """Every other attention instance on the c2 shape: stream-K and clusters of 2/4/6/8."""
    _, res, plan = _run_step("c2", schedule=schedule, sample=16)
    assert plan == schedule
    _assert_ok(res)


def test_c2_page16(cuda_ok, free_gpu):
    _, res, _ = _run_step("c2", page_size=16, sample=16)
    _assert_ok(res)


def test_c3_full_shape(cuda_ok, free_gpu):
    """c3 at 90%: Qwen2.5-7B shapes, 128K x batch 8 (60 GB of target KV), M = 35
    (three 16-row warps, stream-K), long rows through the chunk-parallel select."""
    step, res, plan = _run_step("c3", sample=28)
    assert plan == 1
    assert step._dist is not None
    _assert_ok(res)


def test_c4_single_gpu_sharded_path(cuda_ok, free_gpu):
    """c4 (1M context) at P = 1 through ShardedVerifyStep, exactly as the bench's
    one-GPU c4 point: 137 GB of target KV + 17 GB of draft K."""
    import torch

    from paper_2605_15508_b200 import SparsityConfig, sharded
    from paper_2605_15508_b200.verify_step import config_shape, random_mapping_table

    s = config_shape("c4")
    cfg = SparsityConfig(budget=0.1)
    step = sharded.ShardedVerifyStep(s, cfg, random_mapping_table(s, seed=5), 0, 1, device="cuda", align=64)
    dq, dk, tq, tk, tv = sharded.local_synthetic_inputs(s, step.bounds, 0, "cuda", seed=0)
    dqv, dkv, q, k, v = step.local_views(dq, dk, tq, tk, tv, full=False)
    out, _ = sharded.run_single(step.step(dqv, dkv, q, k, v))
    torch.cuda.synchronize()
    assert step.status.item() == 0
    units = parity.sample_units(s.batch, s.target_layers, s.target_kv_heads, 8, seed=2)
    res = parity.check_units(step, q, k, v, out, units)
    _assert_ok(res)


@pytest.mark.parametrize("schedule", [1, 2, 3, 4, 6, 8])
@pytest.mark.parametrize("gt,gamma", [(4, 4), (7, 4), (1, 4)])
def test_small_shapes_every_schedule(cuda_ok, schedule, gt, gamma):
    """Forced schedules on small shapes across the warp counts (M = 20, 35, 5)."""
    import torch

    from paper_2605_15508_b200 import SparsityConfig
    from paper_2605_15508_b200.verify_step import STSVerifyStep, VerifyShape, random_mapping_table, synthetic_inputs

    s = VerifyShape(batch=2, context=2000, gamma=gamma, target_layers=2, target_q_heads=2 * gt, target_kv_heads=2,
                    head_dim=128, draft_layers=2, draft_q_heads=8, draft_kv_heads=2, draft_head_dim=64)
    step = STSVerifyStep(s, SparsityConfig(budget=0.1), random_mapping_table(s, seed=gt), mode="S",
                         schedule=schedule)
    dq, dk, tq, tk, tv = synthetic_inputs(s, "cuda", seed=gt + schedule)
    q, k, v = step.target_views(tq, tk, tv)
    out, _ = step.step(*step.draft_views(dq, dk), q, k, v)
    torch.cuda.synchronize()
    assert step.status.item() == 0
    res = parity.check_units(step, q, k, v, out, list(range(s.target_units)))
    _assert_ok(res)
