"""TEST INFRASTRUCTURE ONLY — ctypes binding of the CPU oracle (liboracle.so).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference leg may import this package, as the checker or the timed CPU
reference.  The product path (paper_2604_10377_b200) never imports it.

The oracle is a C++ restatement of the reference solver (see
oracle/fmsolve_oracle.cpp for the file:line map).  Parity pinning: the
reference's KATs and golden memory table are replayed in
tests/test_oracle.py; numpy/scipy LAPACK are the independent cross-check.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "liboracle.so"

OK, INVALID_ARGUMENT, SINGULAR, MEMORY_CAP, RANK_DEFICIENT = 0, 1, 2, 3, 5


class Opts(C.Structure):
    _fields_ = [("ridge", C.c_double), ("rcond_threshold", C.c_double), ("has_cap", C.c_int),
                ("cap_bytes", C.c_uint64), ("threads", C.c_uint), ("inject_fault", C.c_int)]


class Report(C.Structure):
    _fields_ = [("max_residual", C.c_double), ("wall_seconds", C.c_double),
                ("peak_extra_bytes", C.c_uint64), ("failing_system", C.c_int64),
                ("required_bytes", C.c_uint64), ("cap_bytes", C.c_uint64),
                ("message", C.c_char * 256)]


class OracleError(Exception):
    def __init__(self, status, report):
        self.status = status
        self.failing_system = report.failing_system if report is not None else -1
        self.required_bytes = report.required_bytes if report is not None else 0
        self.cap_bytes = report.cap_bytes if report is not None else 0
        super().__init__(report.message.decode() if report is not None else f"status {status}")


_lib = None


def build():
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = C.CDLL(str(LIB))
        P, I, I64, D, F = C.c_void_p, C.c_int, C.c_int64, C.c_double, C.c_float
        for name, res, args in [
            ("oracle_solve_f64", I, [I, I64, I, P, P, P, D, C.POINTER(Opts), P, C.POINTER(Report)]),
            ("oracle_solve_f32", I, [I, I64, I, P, P, P, F, C.POINTER(Opts), P, C.POINTER(Report)]),
            ("oracle_solve_full_f64", I, [I, P, P, P, D, D, P, C.POINTER(Report)]),
            ("oracle_solve_full_f32", I, [I, P, P, P, F, F, P, C.POINTER(Report)]),
            ("oracle_mask_f64", I, [I, I, P, P, D, P, C.c_char_p]),
            ("oracle_mask_f32", I, [I, I, P, P, F, P, C.c_char_p]),
            ("oracle_normal_equations", I, [I, I, P, P, P, P]),
            ("oracle_project_mass", I, [I64, I, I, P, P, P, P]),
            ("oracle_residual_f64", D, [I, P, P, P, P, D]),
            ("oracle_energy_f64", D, [I, I, P, P, P, P, D]),
            ("oracle_generate_instance", I, [I, I, C.c_uint64, P, P, P, P]),
            ("oracle_randn", None, [I, I, C.c_uint64, P]),
            ("oracle_hardware_threads", C.c_uint, []),
            ("oracle_rcond_f64", D, [I, P]),
            ("oracle_project_pinv", I, [I64, I, I, P, P, D, P, C.POINTER(C.c_int), C.c_char_p]),
            ("oracle_rcond_f32", F, [I, P]),
        ]:
            fn = getattr(L, name)
            fn.restype, fn.argtypes = res, args
        _lib = L
    return _lib


def _p(a):
    return C.c_void_p(a.ctypes.data)


def _c(a, dt):
    return np.ascontiguousarray(np.asarray(a, dtype=dt))


@dataclass
class SolveResult:
    maps: np.ndarray
    max_residual: float
    wall_seconds: float
    peak_extra_bytes: int


def solve(G, R, M, lam, *, route="batched", dtype=np.float64, ridge=0.0, rcond_threshold=None,
          memory_cap_bytes=None, threads=0, inject_fault=False) -> SolveResult:
    """Reference solver restatement. route: 'rowwise' (solver.hpp:174) or 'batched' (:226).
    G, R, M: [b,k,k] (or [k,k]). Raises OracleError on non-OK status."""
    G = _c(G, dtype)
    single = G.ndim == 2
    if single:
        G, R, M = G[None], _c(R, dtype)[None], _c(M, dtype)[None]
    R, M = _c(R, dtype), _c(M, dtype)
    b, k, _ = G.shape
    out = np.zeros_like(G)
    o = Opts(ridge, -1.0 if rcond_threshold is None else rcond_threshold,
             0 if memory_cap_bytes is None else 1, memory_cap_bytes or 0, threads, int(inject_fault))
    rep = Report()
    fn = lib().oracle_solve_f64 if dtype == np.float64 else lib().oracle_solve_f32
    st = fn(0 if route == "rowwise" else 1, b, k, _p(G), _p(R), _p(M), lam, C.byref(o), _p(out),
            C.byref(rep))
    if st != OK:
        raise OracleError(st, rep)
    return SolveResult(out[0] if single else out, rep.max_residual, rep.wall_seconds,
                       rep.peak_extra_bytes)


def solve_full(G, R, M, lam, ridge=0.0, dtype=np.float64) -> np.ndarray:
    """k^2 x k^2 route (solver.hpp:368-444), dense LU."""
    G, R, M = _c(G, dtype), _c(R, dtype), _c(M, dtype)
    k = G.shape[0]
    out = np.zeros((k, k), dtype)
    rep = Report()
    fn = lib().oracle_solve_full_f64 if dtype == np.float64 else lib().oracle_solve_full_f32
    st = fn(k, _p(G), _p(R), _p(M), lam, ridge, _p(out), C.byref(rep))
    if st != OK:
        raise OracleError(st, rep)
    return out


def mask(kind, ev1, ev2, sigma=0.5, dtype=np.float64) -> np.ndarray:
    """kind: 0 commutativity, 1 resolvent (masks.hpp:13-89)."""
    e1, e2 = _c(ev1, dtype), _c(ev2, dtype)
    if e1.shape != e2.shape:
        raise OracleError(INVALID_ARGUMENT, None)
    k = e1.shape[0]
    out = np.zeros((k, k), dtype)
    msg = C.create_string_buffer(256)
    fn = lib().oracle_mask_f64 if dtype == np.float64 else lib().oracle_mask_f32
    st = fn(int(kind), k, _p(e1), _p(e2), sigma, _p(out), msg)
    if st != OK:
        r = Report()
        r.message = msg.value
        r.failing_system = -1
        raise OracleError(st, r)
    return out


def normal_equations(a, b):
    a, b = _c(a, np.float64), _c(b, np.float64)
    k, d = a.shape
    g, r = np.zeros((k, k)), np.zeros((k, k))
    if lib().oracle_normal_equations(k, d, _p(a), _p(b), _p(g), _p(r)) != OK:
        raise OracleError(INVALID_ARGUMENT, None)
    return g, r


def project_mass(phi, mass, F):
    phi, mass, F = _c(phi, np.float64), _c(mass, np.float64), _c(F, np.float64)
    n, k = phi.shape
    d = F.shape[1]
    out = np.zeros((k, d))
    lib().oracle_project_mass(n, k, d, _p(phi), _p(mass), _p(F), _p(out))
    return out


def residual(C_, G, R, M, lam) -> float:
    C_, G, R, M = (_c(x, np.float64) for x in (C_, G, R, M))
    return lib().oracle_residual_f64(C_.shape[0], _p(C_), _p(G), _p(R), _p(M), lam)


def energy(C_, a, b, M, lam) -> float:
    C_, a, b, M = (_c(x, np.float64) for x in (C_, a, b, M))
    return lib().oracle_energy_f64(a.shape[0], a.shape[1], _p(C_), _p(a), _p(b), _p(M), lam)


def generate_instance(k, d, seed):
    """bench.hpp:52-93 reference generator -> (a, b, ev1, ev2) float64."""
    a, b = np.zeros((k, d)), np.zeros((k, d))
    e1, e2 = np.zeros(k), np.zeros(k)
    lib().oracle_generate_instance(k, d, seed, _p(a), _p(b), _p(e1), _p(e2))
    return a, b, e1, e2


def randn(rows, cols, seed):
    out = np.zeros((rows, cols))
    lib().oracle_randn(rows, cols, seed, _p(out))
    return out


def random_problem(k, d, seed, kind=0, sigma=0.5):
    """test_solver.cpp:25-28: generate_instance + mask -> (G, R, M, a, b)."""
    a, b, e1, e2 = generate_instance(k, d, seed)
    M = mask(kind, e1, e2, sigma)
    G, R = normal_equations(a, b)
    return G, R, M, a, b


def rcond(A, dtype=np.float32) -> float:
    """The reference's rcond estimate of one assembled system A (solver.hpp:158-166:
    PartialPivLU + Hager/Higham); -1 on an exact zero pivot."""
    A = _c(A, dtype)
    fn = lib().oracle_rcond_f64 if dtype == np.float64 else lib().oracle_rcond_f32
    return float(fn(A.shape[0], _p(A)))


def project_pinv(basis, features, condition_threshold=1e10):
    """project_to_spectral (spectral.hpp:47-93) in double: pinv(basis) @ features.
    Raises OracleError(RANK_DEFICIENT) with .rank / .expected on a rank-deficient basis."""
    B, F = _c(basis, np.float64), _c(features, np.float64)
    n, k = B.shape
    d = F.shape[1]
    out = np.zeros((k, d))
    rank = C.c_int(0)
    msg = C.create_string_buffer(256)
    st = lib().oracle_project_pinv(n, k, d, _p(B), _p(F), condition_threshold, _p(out), C.byref(rank), msg)
    if st != OK:
        r = Report()
        r.message = msg.value
        r.failing_system = -1
        err = OracleError(st, r)
        err.rank, err.expected = rank.value, k
        raise err
    return out


def hardware_threads() -> int:
    return int(lib().oracle_hardware_threads())
