"""Python mirror of the reference `fmsolve` solver API, served by libfmap_cuda.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/fmsolve/{solver,masks,types}.hpp so tests read
like the reference's own (proj/tests/test_solver.cpp, test_masks.cpp):

    reference (C++)                          here
    ---------------------------------------  -----------------------------------
    normal_equations(a, b)   solver.hpp:96   normal_equations(a, b)
    make_problem(a, b, mask) solver.hpp:106  make_problem(a, b, mask)
    check_stationarity(...)  solver.hpp:120  check_stationarity(c, a, b, mask, lam)
    solve_batched_many(...)  solver.hpp:226  solve_cuda_many(problems, lam, opts)
    solve_batched(...)       solver.hpp:353  solve_cuda(problem | a, b, mask, lam, opts)
    build_mask(kind, ...)    masks.hpp:85    build_mask(kind, ev1, ev2, sigma=0.5)
    SingularSystemError      types.hpp:25    SingularSystemError (.system())
    MemoryCapExceeded        types.hpp:54    MemoryCapExceeded (.required_bytes(), .cap_bytes())
    std::invalid_argument                    InvalidArgument (a ValueError)

The "cuda" route is a new route: same maps as the reference
routes within the fp32 tolerance, its own peak_extra_bytes accounting (device
staging / scratch bytes, no k^3 term).  Arithmetic is fp32 throughout;
float64 inputs are cast to float32.  Device-tensor entry points
(solve_device, pipeline_device) take torch CUDA tensors and never copy them
to the host.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from datetime import timedelta
from typing import Optional, Sequence

import numpy as np

from . import _lib


# ---------------------------------------------------------------- errors ----
class InvalidArgument(ValueError):
    """std::invalid_argument in the reference."""


class SingularSystemError(RuntimeError):
    """types.hpp:25-36: `system()` is the 0-based global row-system index."""

    def __init__(self, system: int, what: str):
        super().__init__(what)
        self._system = int(system)

    def system(self) -> int:
        return self._system


class RankDeficientError(RuntimeError):
    def __init__(self, rank: int, expected: int, what: str):
        super().__init__(what)
        self._rank, self._expected = rank, expected

    def rank(self) -> int:
        return self._rank

    def expected(self) -> int:
        return self._expected


class MemoryCapExceeded(RuntimeError):
    """types.hpp:54-67: raised before any allocation."""

    def __init__(self, required: int, cap: int, what: str):
        super().__init__(what)
        self._required, self._cap = int(required), int(cap)

    def required_bytes(self) -> int:
        return self._required

    def cap_bytes(self) -> int:
        return self._cap


class CudaError(RuntimeError):
    pass


# ----------------------------------------------------------------- types ----
class MaskKind(enum.Enum):
    Commutativity = _lib.MASK_COMMUTATIVITY
    Resolvent = _lib.MASK_RESOLVENT


def default_rcond_threshold() -> float:
    """solver.hpp:18-27 for Scalar = float."""
    return 1e-7


@dataclass
class SolverOptions:
    """solver.hpp:29-50."""
    ridge: float = 0.0
    rcond_threshold: float = field(default_factory=default_rcond_threshold)
    memory_cap_bytes: Optional[int] = None
    threads: int = 0
    inject_fault: bool = False
    compute_residual: bool = True

    def to_c(self) -> _lib.SolverOptionsC:
        o = _lib.SolverOptionsC()
        o.ridge = float(self.ridge)
        o.rcond_threshold = float(self.rcond_threshold)
        o.has_memory_cap = 0 if self.memory_cap_bytes is None else 1
        o.memory_cap_bytes = int(self.memory_cap_bytes or 0)
        o.threads = int(self.threads)
        o.inject_fault = int(bool(self.inject_fault))
        o.compute_residual = int(bool(self.compute_residual))
        return o


@dataclass
class SolveReport:
    """solver.hpp:52-59."""
    map: np.ndarray
    residual_norm: float = 0.0
    wall_time: timedelta = timedelta(0)
    peak_extra_bytes: int = 0
    min_rcond: float = 0.0
    rcond_exact_systems: int = 0  # systems that needed the exact Hager/Higham estimator


@dataclass
class BatchSolveReport:
    """solver.hpp:61-68; `maps` is a [b, k, k] array (maps[q] is C_q)."""
    maps: object
    max_residual_norm: float = 0.0
    wall_time: timedelta = timedelta(0)
    peak_extra_bytes: int = 0
    min_rcond: float = 0.0
    rcond_exact_systems: int = 0  # systems that needed the exact Hager/Higham estimator


@dataclass
class NormalEquations:
    gram: np.ndarray
    rhs: np.ndarray


@dataclass
class RegularizedProblem:
    neq: NormalEquations
    mask: np.ndarray

    def resolution(self) -> int:
        return int(self.mask.shape[0])


# --------------------------------------------------------------- helpers ----
def _ctx(device: int = 0) -> _lib.Context:
    return _lib.context(device)


def _f32(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.float32))


def _ptr(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data)


def _raise(ctx: _lib.Context, status: int, rep: Optional[_lib.ReportC] = None):
    if status == _lib.FMAP_OK:
        return
    msg = ctx.last_error()
    if status == _lib.FMAP_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if status == _lib.FMAP_SINGULAR:
        raise SingularSystemError(rep.failing_system if rep is not None else -1, msg)
    if status == _lib.FMAP_MEMORY_CAP:
        raise MemoryCapExceeded(rep.required_bytes if rep else 0, rep.cap_bytes if rep else 0, msg)
    if status == _lib.FMAP_RANK_DEFICIENT:
        raise RankDeficientError(-1, -1, msg)
    raise CudaError(f"libfmap_cuda status {status}: {msg}")


def _require(cond: bool, msg: str):
    if not cond:
        raise InvalidArgument(msg)


def _require_finite(a: np.ndarray, name: str):
    if not np.all(np.isfinite(a)):
        raise InvalidArgument(f"{name} contains non-finite entries")


# ----------------------------------------------------------------- masks ----
def build_mask(kind: MaskKind, ev1, ev2, sigma: float = 0.5, device: int = 0) -> np.ndarray:
    """masks.hpp:84-89 (batched when ev1/ev2 are [b, k]); computed on the GPU."""
    e1, e2 = _f32(ev1), _f32(ev2)
    _require(e1.shape == e2.shape, "eigenvalue vectors must have equal length")
    _require(e1.size >= 1, "eigenvalue vectors must be non-empty")
    batched = e1.ndim == 2
    e1b, e2b = (e1, e2) if batched else (e1[None], e2[None])
    b, k = e1b.shape
    out = np.empty((b, k, k), np.float32)
    ctx = _ctx(device)
    st = ctx._lib.fmap_mask_f32(ctx.handle, b, k, _ptr(e1b), _ptr(e2b), int(kind.value),
                                float(sigma), _ptr(out))
    _raise(ctx, st)
    return out if batched else out[0]


def mask_commutativity(ev1, ev2, device: int = 0) -> np.ndarray:
    return build_mask(MaskKind.Commutativity, ev1, ev2, 0.5, device)


def mask_resolvent(ev1, ev2, sigma: float, device: int = 0) -> np.ndarray:
    return build_mask(MaskKind.Resolvent, ev1, ev2, sigma, device)


# ------------------------------------------------------ normal equations ----
def normal_equations(a, b, device: int = 0) -> NormalEquations:
    """solver.hpp:95-103: gram = A A^T, rhs = B A^T (GPU)."""
    A, B = _f32(a), _f32(b)
    _require(A.ndim == 2 and A.shape[0] >= 1 and A.shape[1] >= 1, "descriptor A must be non-empty")
    _require(A.shape == B.shape, "descriptors A and B must have identical shape")
    _require_finite(A, "A")
    _require_finite(B, "B")
    k, d = A.shape
    g = np.empty((k, k), np.float32)
    r = np.empty((k, k), np.float32)
    ctx = _ctx(device)
    st = ctx._lib.fmap_normal_equations_f32(ctx.handle, 1, k, d, _ptr(A), _ptr(B), _ptr(g), _ptr(r))
    _raise(ctx, st)
    return NormalEquations(g, r)


def make_problem(a, b, mask, device: int = 0) -> RegularizedProblem:
    """solver.hpp:105-114."""
    neq = normal_equations(a, b, device)
    M = _f32(mask)
    _require(M.ndim == 2 and M.shape[0] == M.shape[1], "penalty mask must be square")
    _require(M.shape[0] == neq.gram.shape[0], "penalty mask size must match descriptor row count")
    _require_finite(M, "mask")
    _require(bool(np.all(M >= 0)), "penalty mask entries must be non-negative")
    return RegularizedProblem(neq, M)


# ---------------------------------------------------------------- solver ----
def solve_cuda_many(problems: Sequence[RegularizedProblem], lam: float,
                    opts: Optional[SolverOptions] = None, device: int = 0) -> BatchSolveReport:
    """Drop-in for solve_batched_many (solver.hpp:225-322) on the GPU route."""
    opts = opts or SolverOptions()
    _require(len(problems) > 0, "no problems to solve")
    k = problems[0].resolution()
    for p in problems:
        _require(p.mask.ndim == 2 and p.mask.shape[1] == p.mask.shape[0], "penalty mask must be square")
        _require(p.neq.gram.shape == (p.resolution(), p.resolution()), "gram matrix must be k x k")
        _require(p.neq.rhs.shape == (p.resolution(), p.resolution()), "rhs matrix must be k x k")
        _require(p.resolution() == k, "all problems in a batch must share the spectral resolution")
    G = _f32(np.stack([p.neq.gram for p in problems]))
    R = _f32(np.stack([p.neq.rhs for p in problems]))
    M = _f32(np.stack([p.mask for p in problems]))
    return solve_host(G, R, M, lam, opts, device)


def solve_host(G: np.ndarray, R: np.ndarray, M: np.ndarray, lam: float,
               opts: Optional[SolverOptions] = None, device: int = 0,
               precision: str = "f32") -> BatchSolveReport:
    """Host-buffer batched entry: G, R, M are [b, k, k] arrays -> maps [b, k, k].

    precision "f64" selects the f64 route (fmap_solve_f64: the reference's default
    Scalar = double, rcond threshold 1e-14 unless opts sets one)."""
    if precision == "f64":
        opts = opts or SolverOptions(rcond_threshold=-1.0)
        G, R, M = (np.ascontiguousarray(x, dtype=np.float64) for x in (G, R, M))
        _require(G.ndim == 3 and G.shape == R.shape == M.shape and G.shape[1] == G.shape[2],
                 "gram, rhs and mask must be [b, k, k]")
        b, k, _ = G.shape
        out = np.empty((b, k, k), np.float64)
        rep = _lib.ReportC()
        o = opts.to_c()
        if opts.rcond_threshold == default_rcond_threshold():
            o.rcond_threshold = -1.0  # the f32 default was not chosen for f64: use the f64 one (1e-14)
        ctx = _ctx(device)
        st = ctx._lib.fmap_solve_f64(ctx.handle, b, k, _ptr(G), _ptr(R), _ptr(M), float(lam), C.byref(o),
                                     _ptr(out), C.byref(rep))
        _raise(ctx, st, rep)
        return BatchSolveReport(out, rep.max_residual, timedelta(seconds=rep.wall_seconds),
                                int(rep.peak_extra_bytes), rep.min_rcond, int(rep.rcond_exact_systems))
    _require(precision == "f32", "precision must be 'f32' or 'f64'")
    opts = opts or SolverOptions()
    G, R, M = _f32(G), _f32(R), _f32(M)
    _require(G.ndim == 3 and G.shape == R.shape == M.shape and G.shape[1] == G.shape[2],
             "gram, rhs and mask must be [b, k, k]")
    b, k, _ = G.shape
    out = np.empty((b, k, k), np.float32)
    rep = _lib.ReportC()
    o = opts.to_c()
    ctx = _ctx(device)
    st = ctx._lib.fmap_solve_f32(ctx.handle, b, k, _ptr(G), _ptr(R), _ptr(M), float(lam),
                                 C.byref(o), _ptr(out), C.byref(rep))
    _raise(ctx, st, rep)
    return BatchSolveReport(out, rep.max_residual, timedelta(seconds=rep.wall_seconds),
                            int(rep.peak_extra_bytes), rep.min_rcond, int(rep.rcond_exact_systems))


def solve_cuda(problem_or_a, *args, device: int = 0, **kw) -> SolveReport:
    """solve_batched(problem, lam, opts) or solve_batched(a, b, mask, lam, opts)
    (solver.hpp:352-366), through the GPU route."""
    if isinstance(problem_or_a, RegularizedProblem):
        problem = problem_or_a
        lam, *rest = args
    else:
        b_desc, mask, lam, *rest = args
        problem = make_problem(problem_or_a, b_desc, mask, device)
    opts = rest[0] if rest else kw.get("opts")
    batch = solve_cuda_many([problem], lam, opts, device)
    return SolveReport(batch.maps[0], batch.max_residual_norm, batch.wall_time,
                       batch.peak_extra_bytes, batch.min_rcond, batch.rcond_exact_systems)


# Drop-in aliases: the reference names of the one-dispatch route.
solve_batched_many = solve_cuda_many
solve_batched = solve_cuda


def project_to_spectral(basis, features, condition_threshold: float = 1e10, device: int = 0,
                        precision: str = "f64") -> np.ndarray:
    """spectral.hpp:47-93 on the GPU: pinv(basis) @ features for one basis [n, k]
    or a batch [b, n, k] (features [.., n, d]).  Raises RankDeficientError
    (rank(), expected()) like the reference; InvalidArgument on bad input."""
    B = np.asarray(basis)
    Fm = np.asarray(features)
    single = B.ndim == 2
    if single:
        B, Fm = B[None], Fm[None]
    _require(B.ndim == 3 and B.shape[1] >= 1 and B.shape[2] >= 1, "basis must be non-empty")
    _require(Fm.ndim == 3 and Fm.shape[2] >= 1 and Fm.shape[1] >= 1, "features must be non-empty")
    if Fm.shape[1] != B.shape[1]:
        raise InvalidArgument(f"feature row count ({Fm.shape[1]}) does not match basis vertex count ({B.shape[1]})")
    _require(Fm.shape[0] == B.shape[0], "one feature matrix per basis")
    b, n, k = B.shape
    d = Fm.shape[2]
    dt = np.float64 if precision == "f64" else np.float32
    B = np.ascontiguousarray(B, dtype=dt)
    Fm = np.ascontiguousarray(Fm, dtype=dt)
    out = np.zeros((b, k, d), dt)
    ranks = np.zeros(b, np.int64)
    ctx = _ctx(device)
    rep = _lib.ReportC()
    fn = ctx._lib.fmap_project_pinv_f64 if precision == "f64" else ctx._lib.fmap_project_pinv_f32
    st = fn(ctx.handle, b, n, k, d, _ptr(B), _ptr(Fm), float(condition_threshold), _ptr(out), _ptr(ranks),
            C.byref(rep))
    if st == _lib.FMAP_RANK_DEFICIENT:
        q = int(rep.failing_system)
        raise RankDeficientError(int(ranks[q]), k, ctx.last_error())
    _raise(ctx, st, rep)
    return out[0] if single else out


def check_stationarity(c, a, b, mask, lam: float, device: int = 0) -> float:
    """solver.hpp:116-128: ||C AA^T + lambda (M .* C) - BA^T||_F (GPU, fp64 accumulation)."""
    import torch  # device plumbing only
    problem = make_problem(a, b, mask, device)
    _require(lam >= 0, "lambda must be non-negative")
    Cm = _f32(c)
    _require(Cm.shape == problem.mask.shape, "map C must match the penalty mask shape")
    dev = torch.device("cuda", device)
    t = [torch.from_numpy(x).to(dev)[None].contiguous()
         for x in (Cm, problem.neq.gram, problem.neq.rhs, problem.mask)]
    out = torch.empty(1, dtype=torch.float64, device=dev)
    ctx = _ctx(device)
    ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
    try:
        st = ctx._lib.fmap_residual_f32_dev(ctx.handle, 1, Cm.shape[0], *(C.c_void_p(x.data_ptr()) for x in t),
                                            float(lam), C.c_void_p(out.data_ptr()))
        _raise(ctx, st)
        return float(out.item())
    finally:
        ctx.set_stream(None)


# ------------------------------------------------------ device-tensor API ----
def _dptr(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr())


def _check_dev(t, name, shape=None):
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
        raise InvalidArgument(f"{name} must be a contiguous float32 CUDA tensor")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise InvalidArgument(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")


def solve_device(gram, rhs, mask=None, *, lam: float, ev1=None, ev2=None,
                 mask_kind: MaskKind = MaskKind.Resolvent, sigma: float = 0.5,
                 opts: Optional[SolverOptions] = None, out=None):
    """Batched solve on torch CUDA tensors ([b,k,k]); returns (C, BatchSolveReport).

    Pass `mask` for the reference contract, or `ev1`/`ev2` ([b,k]) to generate the
    mask rows inside the solver (fused; M never touches HBM)."""
    import torch
    opts = opts or SolverOptions()
    _check_dev(gram, "gram")
    b, k, _ = gram.shape
    _check_dev(rhs, "rhs", (b, k, k))
    if out is None:
        out = torch.empty_like(gram)
    _check_dev(out, "out", (b, k, k))
    dev = gram.device.index or 0
    ctx = _ctx(dev)
    ctx.set_stream(torch.cuda.current_stream(gram.device).cuda_stream)
    rep = _lib.ReportC()
    o = opts.to_c()
    try:
        if mask is not None:
            _check_dev(mask, "mask", (b, k, k))
            st = ctx._lib.fmap_solve_f32_dev(ctx.handle, b, k, _dptr(gram), _dptr(rhs), _dptr(mask),
                                             float(lam), C.byref(o), _dptr(out), C.byref(rep))
        else:
            _check_dev(ev1, "ev1", (b, k))
            _check_dev(ev2, "ev2", (b, k))
            st = ctx._lib.fmap_solve_ev_f32_dev(ctx.handle, b, k, _dptr(gram), _dptr(rhs), _dptr(ev1),
                                                _dptr(ev2), int(mask_kind.value), float(sigma),
                                                float(lam), C.byref(o), _dptr(out), C.byref(rep))
        _raise(ctx, st, rep)
    finally:
        ctx.set_stream(None)
    return out, BatchSolveReport(out, rep.max_residual, timedelta(seconds=rep.wall_seconds),
                                 int(rep.peak_extra_bytes), rep.min_rcond, int(rep.rcond_exact_systems))


def pipeline_device(phi1, mass1, F1, ev1, phi2, mass2, F2, ev2, *, lam: float = 100.0,
                    sigma: float = 0.5, mask_kind: MaskKind = MaskKind.Resolvent,
                    bidirectional: bool = False, opts: Optional[SolverOptions] = None):
    """(Phi, Mass, F, ev) x 2 -> C_xy (and C_yx) on the GPU.  Shapes:
    phi [b,n,k], mass [b,n], F [b,n,d], ev [b,k] (n may differ per side)."""
    import torch
    opts = opts or SolverOptions()
    for t, nm in ((phi1, "phi1"), (mass1, "mass1"), (F1, "F1"), (ev1, "ev1"),
                  (phi2, "phi2"), (mass2, "mass2"), (F2, "F2"), (ev2, "ev2")):
        _check_dev(t, nm)
    b, n1, k = phi1.shape
    n2 = phi2.shape[1]
    d = F1.shape[2]
    _require(tuple(phi2.shape) == (b, n2, k), "phi2 shape mismatch")
    _require(tuple(F1.shape) == (b, n1, d) and tuple(F2.shape) == (b, n2, d), "feature shape mismatch")
    _require(tuple(mass1.shape) == (b, n1) and tuple(mass2.shape) == (b, n2), "mass shape mismatch")
    _require(tuple(ev1.shape) == (b, k) and tuple(ev2.shape) == (b, k), "eigenvalue shape mismatch")
    cxy = torch.empty((b, k, k), device=phi1.device, dtype=torch.float32)
    cyx = torch.empty_like(cxy) if bidirectional else None
    ctx = _ctx(phi1.device.index or 0)
    ctx.set_stream(torch.cuda.current_stream(phi1.device).cuda_stream)
    rep = _lib.ReportC()
    o = opts.to_c()
    try:
        st = ctx._lib.fmap_pipeline_f32_dev(
            ctx.handle, b, n1, n2, k, d, _dptr(phi1), _dptr(mass1), _dptr(F1), _dptr(ev1),
            _dptr(phi2), _dptr(mass2), _dptr(F2), _dptr(ev2), int(mask_kind.value), float(sigma),
            float(lam), C.byref(o), _dptr(cxy), _dptr(cyx) if cyx is not None else C.c_void_p(0),
            C.byref(rep))
        _raise(ctx, st, rep)
    finally:
        ctx.set_stream(None)
    return cxy, cyx, BatchSolveReport(cxy, rep.max_residual, timedelta(seconds=rep.wall_seconds),
                                      int(rep.peak_extra_bytes), rep.min_rcond, int(rep.rcond_exact_systems))
