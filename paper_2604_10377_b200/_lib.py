"""ctypes binding of libfmap_cuda.so (include/fmap_cuda.h).

There is no CPU fallback: if the shared library is missing or no CUDA device
is present, every compute entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libfmap_cuda.so"
if os.environ.get("FMAP_LIB_VARIANT"):  # developer A/B: a second in-tree build, libfmap_cuda_<v>.so
    LIB_PATH = LIB_PATH.with_name(f"libfmap_cuda_{os.environ['FMAP_LIB_VARIANT']}.so")

FMAP_OK = 0
FMAP_INVALID_ARGUMENT = 1
FMAP_SINGULAR = 2
FMAP_MEMORY_CAP = 3
FMAP_CUDA_ERROR = 4
FMAP_RANK_DEFICIENT = 5

MASK_COMMUTATIVITY = 0
MASK_RESOLVENT = 1

# Every symbol include/fmap_cuda.h declares (checked by tests/test_abi.py).
EXPORTED = [
    "fmap_ctx_create", "fmap_ctx_destroy", "fmap_ctx_set_stream", "fmap_last_error",
    "fmap_abi_version", "fmap_default_options", "fmap_solve_f32", "fmap_solve_f32_dev",
    "fmap_solve_ev_f32_dev", "fmap_mask_f32", "fmap_mask_f32_dev",
    "fmap_normal_equations_f32", "fmap_normal_equations_f32_dev", "fmap_project_f32_dev",
    "fmap_residual_f32_dev", "fmap_pipeline_f32_dev", "fmap_max_resolution",
    "fmap_last_launch_count", "fmap_last_launches", "fmap_solve_f64", "fmap_solve_f64_dev",
    "fmap_project_pinv_f64", "fmap_project_pinv_f64_dev", "fmap_project_pinv_f32",
]


class SolverOptionsC(C.Structure):
    _fields_ = [
        ("ridge", C.c_float),
        ("rcond_threshold", C.c_float),
        ("has_memory_cap", C.c_int),
        ("memory_cap_bytes", C.c_uint64),
        ("threads", C.c_uint),
        ("inject_fault", C.c_int),
        ("compute_residual", C.c_int),
    ]


class ReportC(C.Structure):
    _fields_ = [
        ("max_residual", C.c_double),
        ("wall_seconds", C.c_double),
        ("peak_extra_bytes", C.c_uint64),
        ("failing_system", C.c_int64),
        ("required_bytes", C.c_uint64),
        ("cap_bytes", C.c_uint64),
        ("min_rcond", C.c_double),
        ("rcond_exact_systems", C.c_int64),
        ("factor_seconds", C.c_double),
    ]


_lib = None
_lock = threading.Lock()


def load() -> C.CDLL:
    """Load (once) the CUDA library; raise if it was not built."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2604_10377_b200.build` "
                "(there is no CPU fallback)")
        lib = C.CDLL(str(LIB_PATH))
        P, I64, F, I = C.c_void_p, C.c_int64, C.c_float, C.c_int
        opt, rep = C.POINTER(SolverOptionsC), C.POINTER(ReportC)
        sig = {
            "fmap_ctx_create": (I, [I, C.POINTER(P)]),
            "fmap_ctx_destroy": (I, [P]),
            "fmap_ctx_set_stream": (I, [P, P]),
            "fmap_last_error": (C.c_char_p, [P]),
            "fmap_abi_version": (I, []),
            "fmap_default_options": (None, [opt]),
            "fmap_solve_f32": (I, [P, I64, I64, P, P, P, F, opt, P, rep]),
            "fmap_solve_f32_dev": (I, [P, I64, I64, P, P, P, F, opt, P, rep]),
            "fmap_solve_f64": (I, [P, I64, I64, P, P, P, C.c_double, opt, P, rep]),
            "fmap_solve_f64_dev": (I, [P, I64, I64, P, P, P, C.c_double, opt, P, rep]),
            "fmap_solve_ev_f32_dev": (I, [P, I64, I64, P, P, P, P, I, F, F, opt, P, rep]),
            "fmap_mask_f32": (I, [P, I64, I64, P, P, I, F, P]),
            "fmap_mask_f32_dev": (I, [P, I64, I64, P, P, I, F, P]),
            "fmap_normal_equations_f32": (I, [P, I64, I64, I64, P, P, P, P]),
            "fmap_normal_equations_f32_dev": (I, [P, I64, I64, I64, P, P, P, P]),
            "fmap_project_f32_dev": (I, [P, I64, I64, I64, I64, P, P, P, P]),
            "fmap_residual_f32_dev": (I, [P, I64, I64, P, P, P, P, F, P]),
            "fmap_pipeline_f32_dev": (I, [P, I64, I64, I64, I64, I64, P, P, P, P, P, P, P, P,
                                          I, F, F, opt, P, P, rep]),
            "fmap_max_resolution": (I64, [P]),
            "fmap_last_launch_count": (I64, [P]),
            "fmap_last_launches": (C.c_char_p, [P]),
            "fmap_project_pinv_f64": (I, [P, I64, I64, I64, I64, P, P, C.c_double, P, P, rep]),
            "fmap_project_pinv_f64_dev": (I, [P, I64, I64, I64, I64, P, P, C.c_double, P, P, rep]),
            "fmap_project_pinv_f32": (I, [P, I64, I64, I64, I64, P, P, F, P, P, rep]),
        }
        for name, (res, args) in sig.items():
            if os.environ.get("FMAP_LIB_VARIANT") and not hasattr(lib, name):
                continue  # developer A/B against an older build
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def exported_symbols() -> list[str]:
    """Names the library actually exports (for the CPU-side ABI test)."""
    lib = C.CDLL(str(LIB_PATH))
    return [n for n in EXPORTED if hasattr(lib, n)]


class Context:
    """One device + stream + grow-only device arena (BatchedWorkspace analogue)."""

    def __init__(self, device: int = 0):
        lib = load()
        h = C.c_void_p()
        st = lib.fmap_ctx_create(int(device), C.byref(h))
        if st != FMAP_OK:
            raise RuntimeError(f"fmap_ctx_create(device={device}) failed with status {st} "
                               "(no CUDA device? there is no CPU fallback)")
        self._lib = lib
        self.handle = h
        self.device = device

    def close(self):
        if getattr(self, "handle", None):
            self._lib.fmap_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def last_error(self) -> str:
        return self._lib.fmap_last_error(self.handle).decode()

    def set_stream(self, stream_ptr: int | None):
        self._lib.fmap_ctx_set_stream(self.handle, C.c_void_p(stream_ptr or 0))

    @property
    def max_resolution(self) -> int:
        return int(self._lib.fmap_max_resolution(self.handle))

    @property
    def last_launch_count(self) -> int:
        return int(self._lib.fmap_last_launch_count(self.handle))

    @property
    def last_launches(self) -> list[str]:
        """Kernel names the last call launched, in order (fmap_last_launches)."""
        names = self._lib.fmap_last_launches(self.handle).decode()
        return names.split(",") if names else []


_contexts: dict[int, Context] = {}


def context(device: int = 0) -> Context:
    ctx = _contexts.get(device)
    if ctx is None:
        ctx = Context(device)
        _contexts[device] = ctx
    return ctx
