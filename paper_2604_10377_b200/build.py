"""Build libfmap_cuda.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2604_10377_b200.build

The shared library lands next to this file so it travels with the repo
snapshot to the GPU box (it is git-ignored, not gpurun-ignored).
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
ROOT = PKG.parent
LIB = PKG / "libfmap_cuda.so"
SOURCES = ["fmap_tc.cu", "fmap_gram.cu", "fmap_f64.cu", "fmap_pinv.cu", "fmap_kernels.cu", "fmap_capi.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "fmap_cuda.h"]
    objdir = PKG / "_build"
    objdir.mkdir(exist_ok=True)
    stamp = objdir / "flags.txt"  # a change of FMAP_NVCC_FLAGS rebuilds every object
    flags = os.environ.get("FMAP_NVCC_FLAGS", "")
    if not stamp.exists() or stamp.read_text() != flags:
        force = True
        stamp.write_text(flags)
    if not force and not _stale(LIB, deps):
        return LIB
    common = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-I", str(ROOT / "include"), "-Xptxas", "-v",
              *os.environ.get("FMAP_NVCC_FLAGS", "").split()]  # e.g. -DFMAP_TC_TRACE (phase stamps)
    def compile_one(src: str) -> str:
        obj = objdir / (Path(src).stem + ".o")
        if not force and not _stale(obj, [CSRC / src, *CSRC.glob("*.cuh"), ROOT / "include" / "fmap_cuda.h"]):
            return str(obj)
        cmd = [*common, "-c", str(CSRC / src), "-o", str(obj)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(res.stderr)
        return str(obj)

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as pool:
        objs = list(pool.map(compile_one, SOURCES))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), *ARCH, "-shared", "-o", str(tmp), *objs, "-cudart", "static"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, LIB)
    return LIB


def build_oracle() -> Path:
    """Compile the CPU checker (test infrastructure, oracle/)."""
    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle")], check=True)
    return ROOT / "oracle" / "_build" / "liboracle.so"


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
    print(build_oracle())
