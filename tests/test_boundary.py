"""CPU-only checks of the drop-in boundary: the C-ABI library loads and
exports exactly what include/sts_b200.h declares, status codes map to the
reference exception classes, and the host-side config / table logic matches
the reference (no kernel launches: there is no GPU here)."""

import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT


def _header_symbols():
    text = (ROOT / "include" / "sts_b200.h").read_text()
    return set(re.findall(r"^STS_API\s+[\w\s\*]+?\b(sts_\w+)\s*\(", text, flags=re.M))


def test_library_builds_and_exports_header_symbols():
    from paper_2605_15508_b200 import _lib
    from paper_2605_15508_b200.build import build

    lib_path = build()
    lib = _lib.load()
    declared = _header_symbols()
    assert len(declared) >= 12
    assert declared == set(_lib.SIGNATURES), "ctypes table and header disagree"
    nm = subprocess.run(["nm", "-D", "--defined-only", str(lib_path)], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (sts_\w+)", nm))
    assert declared <= exported, f"missing exports: {declared - exported}"
    assert lib.sts_abi_version() == _lib.ABI_VERSION == 8
    assert lib.sts_dist_select_bins() == _lib.STS_DIST_BINS


def test_status_codes_map_to_reference_exceptions():
    from paper_2605_15508_b200.errors import (ConfigError, ContractViolation, DeviceError, InputError,
                                              raise_for_status)

    raise_for_status(0, "")
    with pytest.raises(ConfigError):
        raise_for_status(1, "bad budget")
    assert issubclass(ConfigError, InputError)
    with pytest.raises(ContractViolation):
        raise_for_status(2, "empty mask")
    with pytest.raises(DeviceError):
        raise_for_status(3, "cuda")


def test_host_validation_without_gpu():
    """Argument validation happens on the host side of the ABI and reports
    through sts_last_error, so it is testable without a device."""
    from paper_2605_15508_b200 import _lib
    from paper_2605_15508_b200.errors import ConfigError, ContractViolation

    with pytest.raises(ConfigError, match="fractional budget"):
        _lib.call("sts_select_topk", 8, 4, None, 1, 1, None, 4, 1.5, 1, 1, 0, 0, 0, 8, 4, 8, None,
                  None, 0, None)
    with pytest.raises(ConfigError, match="page_size"):
        _lib.call("sts_select_topk", 8, 4, None, 1, 1, None, 4, 2.0, 0, 0, 0, 0, 0, 8, 4, 8, None,
                  None, 0, None)
    with pytest.raises(ContractViolation, match="nsrc"):
        _lib.call("sts_select_topk", 8, 4, None, 3, 1, None, 4, 2.0, 0, 1, 0, 0, 0, 8, 4, 8, None,
                  None, 0, None)
    with pytest.raises(ContractViolation, match="membership"):
        _lib.call("sts_sparse_decode", 1, 1, 8, 8, 8, 64, 0, 1, 40, 64, 8, 4, 8, 0, 8, -1, 1, 0, 0.125, 8,
                  None, 1, None, None, 0, None)
    with pytest.raises(ContractViolation, match="out_dtype"):
        _lib.call("sts_sparse_decode", 0, 1, 8, 8, 8, 64, 0, 1, 4, 64, 8, 4, 8, 0, None, -1, 1, 0, 0.125, 8,
                  None, 1, None, None, 0, None)
    # sharded selection: geometry checked before any launch
    g = _lib.DistRows(8, 64, None, 1, 4, 100, 3, 32, 10, 2)
    import ctypes
    with pytest.raises(ContractViolation, match="page-aligned"):
        _lib.call("sts_dist_select_begin", ctypes.addressof(g), 8, 8, 1 << 30, None)
    g = _lib.DistRows(8, 64, None, 1, 4, 100, 0, 32, 10, 1)
    with pytest.raises(ContractViolation, match="workspace too small"):
        _lib.call("sts_dist_select_begin", ctypes.addressof(g), 8, 8, 16, None)
    g = _lib.DistRows(8, 64, None, 1, 4, 100, 0, 32, 0, 1)
    with pytest.raises(ConfigError, match="k must be"):
        _lib.call("sts_dist_select_begin", ctypes.addressof(g), 8, 8, 1 << 30, None)
    lib = _lib.load()
    assert lib.sts_dist_select_rounds(1) == 3 and lib.sts_dist_select_rounds(16) == 6
    assert lib.sts_dist_select_workspace_bytes(256, 131072, 1) >= 256 * 131072 * 4
    # the oracle's restatement of the protocol uses the same digits (top-down,
    # widths <= STS_DIST_BINS bins, covering every key bit once)
    from oracle.sts_oracle import dist_digits

    for kbits, ps in ((32, 1), (64, 16)):
        dg = dist_digits(kbits)
        assert len(dg) == lib.sts_dist_select_rounds(ps)
        assert sum(w for _, w in dg) == kbits and dg[-1][0] == 0
        assert all(1 << w <= _lib.STS_DIST_BINS for _, w in dg)
        assert [sh for sh, _ in dg] == sorted((sh for sh, _ in dg), reverse=True)


def test_sparsity_config_mirrors_reference():
    from paper_2605_15508_b200 import ConfigError, SparsityConfig

    # pkg/tests/test_sparsity.py:269-289
    with pytest.raises(ConfigError):
        SparsityConfig(budget=1.5)
    with pytest.raises(ConfigError):
        SparsityConfig(budget=0)
    with pytest.raises(ConfigError):
        SparsityConfig(budget=4, scope="sometimes")
    cfg = SparsityConfig(budget=1 / 8)
    assert cfg.tokens_for_context(64) == 8
    assert cfg.tokens_for_context(3) == 1
    assert SparsityConfig(budget=1.0).tokens_for_context(7) == 7
    assert SparsityConfig(budget=0.1).tokens_for_context(32769) == 3277


def test_index_capacity_bounds_selection_sizes():
    from oracle import sts_oracle as O
    from paper_2605_15508_b200.kernels import index_capacity

    rng = np.random.default_rng(0)
    for _ in range(200):
        n = int(rng.integers(1, 600))
        budget = float(rng.choice([0.1, 0.02, 0.5, 1.0])) if rng.random() < 0.5 else int(rng.integers(1, 50))
        ps = int(rng.choice([1, 2, 4, 16]))
        cur, sink, win = bool(rng.random() < 0.5), bool(rng.random() < 0.5), int(rng.integers(0, 9))
        row = rng.random(n).astype(np.float32)
        got = O.select_row(row, O.OracleSparsityConfig(budget, ps, cur, sink, win))
        assert got.size <= index_capacity(n, budget, ps, cur, sink, win)


def test_mapping_table_and_nearest():
    from paper_2605_15508_b200 import HeadMapping, MappingSet

    entries = {(l, h): ((l // 2, (h + l) % 4), 0) for l in range(4) for h in range(8)}
    m = HeadMapping(410, entries)
    t = m.to_table(4, 8, 4)
    assert t.shape == (4, 8) and t[3, 5] == (3 // 2) * 4 + (5 + 3) % 4
    ms = MappingSet([HeadMapping(8, {}), HeadMapping(16, {}), HeadMapping(12, {})])
    # src/headmap.py:181-182: ties -> smaller k
    assert ms.nearest(10).k == 8 and ms.nearest(14).k == 12 and ms.nearest(100).k == 16


def test_verify_shapes_and_algorithmic_bytes():
    from paper_2605_15508_b200.verify_step import algorithmic_bytes, config_shape

    s = config_shape("c2")
    assert s.target_units == 256 and s.rows == 5 and s.target_group == 4
    b = algorithmic_bytes(s, 3277 + 5)
    # ~435.5 MB sparse bytes per verify step at c2
    assert 430e6 < b < 440e6
    dense = algorithmic_bytes(s, s.n_kv, dense=True)
    assert 4.2e9 < dense < 4.4e9
