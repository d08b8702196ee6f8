"""compute-sanitizer over small invocations of every kernel family
(tools/sanitize_run.py): memcheck (out-of-bounds / misaligned accesses),
racecheck (shared-memory hazards: cp.async rings, DSMEM cluster exchanges),
synccheck (barrier misuse) — SURVEY §5 row 2."""

import os
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool,parts", [
    ("memcheck", []),
    ("racecheck", ["select", "decode", "dist", "merge", "prefill", "block", "union"]),
    ("racecheck", ["capture"]),
    ("racecheck", ["prefill_tc", "offload"]),
    ("synccheck", []),
])
def test_sanitizer_clean(cuda_ok, tool, parts):
    if not Path(SAN).exists():
        pytest.skip("compute-sanitizer not found")
    cmd = [SAN, "--tool", tool, "--error-exitcode", "7", "--print-limit", "20", sys.executable,
           str(ROOT / "tools" / "sanitize_run.py"), *parts]
    env = dict(os.environ, PYTORCH_NO_CUDA_MEMORY_CACHING="1")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=str(ROOT))
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, f"{tool} reported errors (rc {r.returncode}):\n{tail}"
    assert "sanitize_run ok" in r.stdout
    text = r.stdout + r.stderr
    assert "ERROR SUMMARY: 0 errors" in text or "SUMMARY: 0 hazards displayed (0 errors, 0 warnings)" in text, tail
