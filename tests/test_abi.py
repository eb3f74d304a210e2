"""C-ABI boundary checks that need no GPU: the library loads, exports every
function include/fmap_cuda.h declares, and the C++ adapter
(include/fmsolve_cuda.hpp) compiles and links against it."""
import ctypes
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "fmap_cuda.h"


def declared_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(fmap_[a-z0-9_]+)\s*\(", text)))


def test_library_exists_and_is_sm100a():
    from paper_2604_10377_b200 import _lib
    assert _lib.LIB_PATH.exists(), "run python -m paper_2604_10377_b200.build"
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_every_declared_symbol_is_exported():
    from paper_2604_10377_b200 import _lib
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    names = declared_functions()
    assert len(names) >= 18
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) == set(_lib.EXPORTED)


def test_abi_version_and_defaults_without_gpu():
    from paper_2604_10377_b200 import _lib
    lib = _lib.load()
    assert lib.fmap_abi_version() == 1
    o = _lib.SolverOptionsC()
    lib.fmap_default_options(ctypes.byref(o))
    assert o.rcond_threshold < 0 and o.compute_residual == 1 and o.inject_fault == 0


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2604_10377_b200 import _lib
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.Context(0)


def test_cpp_adapter_compiles_and_links(tmp_path):
    exe = tmp_path / "test_adapter"
    cmd = ["g++", "-std=c++20", "-O1", "-I", str(ROOT / "include"), str(ROOT / "tests/cpp/test_adapter.cpp"),
           "-L", str(ROOT / "paper_2604_10377_b200"), "-lfmap_cuda",
           f"-Wl,-rpath,{ROOT / 'paper_2604_10377_b200'}", "-o", str(exe)]
    subprocess.run(cmd, check=True)
    rc = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert rc.returncode in (0, 77), rc.stdout + rc.stderr
