import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def unpack(data, offs):
    return [data[offs[i] : offs[i + 1]] for i in range(len(offs) - 1)]


def load_golden(name):
    z = np.load(GOLDEN / name, allow_pickle=False)
    return {k: z[k] for k in z.files}


def cfg_from_json(entry):
    """[budget, is_int, page_size, include_current, include_sink, recent_window]."""
    budget, is_int, ps, cur, sink, win = entry
    budget = int(budget) if is_int else float(budget)
    return budget, ps, cur, sink, win


@pytest.fixture(scope="session")
def cuda_ok():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True
