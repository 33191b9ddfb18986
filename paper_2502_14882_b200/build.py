"""Build the CUDA product library in-tree: paper_2502_14882_b200/libkvq_b200.so.

nvcc for sm_100a only (`-gencode arch=compute_100a,code=sm_100a`), -lineinfo for ncu
source mapping, no fast-math (K1 codes must be bit-exact).
Incremental: a translation unit is recompiled when it or any header is newer than its
object file.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
# KVQ_BUILD_VARIANT=name (experiments only): objects in build_<name>/, library
# libkvq_b200_<name>.so, loaded with KVQ_LIB_PATH - the product library is untouched.
_VARIANT = os.environ.get("KVQ_BUILD_VARIANT", "")
OBJ = PKG / (f"build_{_VARIANT}" if _VARIANT else "build")
LIB = PKG / (f"libkvq_b200_{_VARIANT}.so" if _VARIANT else "libkvq_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", f"-I{ROOT / 'include'}", f"-I{CSRC}"]
# Debug builds only (e.g. KVQ_NVCC_EXTRA=-DKVQ_TRACE_BLOCKS for per-block decode timelines).
FLAGS += os.environ.get("KVQ_NVCC_EXTRA", "").split()


def _headers() -> list[Path]:
    return list(CSRC.glob("*.cuh")) + list((ROOT / "include").glob("*.h"))


def _compile(src: Path, verbose: bool) -> Path:
    obj = OBJ / (src.stem + ".o")
    newest = max([src.stat().st_mtime] + [h.stat().st_mtime for h in _headers()])
    if obj.exists() and obj.stat().st_mtime >= newest:
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, "-c", str(src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed on {src.name}")
    (OBJ / (src.stem + ".ptxas.txt")).write_text(res.stderr)
    if verbose:
        print(f"[build] compiled {src.name}")
    return obj


def build(verbose: bool = True) -> Path:
    OBJ.mkdir(exist_ok=True)
    sources = sorted(CSRC.glob("*.cu"))
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), sources))
    if not LIB.exists() or LIB.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lcudart"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("link failed")
        if verbose:
            print(f"[build] linked {LIB.relative_to(ROOT)}")
    return LIB


if __name__ == "__main__":
    build()
