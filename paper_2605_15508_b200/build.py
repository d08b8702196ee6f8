"""Build libsts_b200.so (sm_100a) in-tree with nvcc.

    python -m paper_2605_15508_b200.build [--force]

The library is plain C-ABI (include/sts_b200.h); Python binds it with ctypes,
so there is no torch extension to JIT and the .so travels with the repo.
"""

from __future__ import annotations

import argparse
import hashlib
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "_lib"
LIB = LIBDIR / "libsts_b200.so"
STAMP = LIBDIR / "libsts_b200.sha"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-O2,-fvisibility=hidden",
    "-Xptxas", "-O3",
    "-shared",
]


def _sources():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "sts_b200.h"]


def _digest() -> str:
    h = hashlib.sha256()
    for p in _sources():
        h.update(p.name.encode())
        h.update(p.read_bytes())
    h.update(" ".join(NVCC_FLAGS).encode())
    return h.hexdigest()


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: cannot build libsts_b200.so")


def _compile_all(out: Path, extra: list[str], verbose: bool = False) -> None:
    """nvcc every .cu to an object in parallel (one process per file), then link."""
    from concurrent.futures import ThreadPoolExecutor

    objdir = LIBDIR / "obj" / out.stem
    objdir.mkdir(parents=True, exist_ok=True)
    cflags = [f for f in NVCC_FLAGS if f != "-shared"]
    srcs = sorted(CSRC.glob("*.cu"))

    def one(src: Path) -> Path:
        obj = objdir / (src.stem + ".o")
        cmd = [nvcc_path(), *cflags, *extra, "-c", "-o", str(obj), str(src)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
        return obj

    with ThreadPoolExecutor(max_workers=max(1, min(len(srcs), os.cpu_count() or 1))) as ex:
        objs = list(ex.map(one, srcs))
    subprocess.run([nvcc_path(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(out),
                    *[str(o) for o in objs]], check=True)


def build_variant(name: str, defines: list[str]) -> Path:
    """Tuning aid: build a copy of the library with extra -D flags into
    _lib/variants/libsts_b200_<name>.so (select it with STS_B200_LIB)."""
    out = LIBDIR / "variants" / f"libsts_b200_{name}.so"
    out.parent.mkdir(parents=True, exist_ok=True)
    _compile_all(out, [f"-D{d}" for d in defines])
    return out


def build(force: bool = False, verbose: bool = False) -> Path:
    digest = _digest()
    if LIB.exists() and STAMP.exists() and STAMP.read_text().strip() == digest and not force:
        return LIB
    LIBDIR.mkdir(exist_ok=True)
    tmp = LIBDIR / "libsts_b200.so.tmp"
    _compile_all(tmp, [], verbose)
    tmp.replace(LIB)
    STAMP.write_text(digest)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose))
