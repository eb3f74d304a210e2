"""B200-native (sm_100a) batched regularized functional-map solver.

Drop-in for the solver path of the reference `fmsolve` library
(/root/reference/proj/include/fmsolve/solver.hpp, masks.hpp): the C ABI is
include/fmap_cuda.h (libfmap_cuda.so, built in-tree for sm_100a), the C++
adapter with the reference signatures is include/fmsolve_cuda.hpp, and this
package mirrors the same API in Python (fmsolve.py).
"""
from ._lib import LIB_PATH, load  # noqa: F401
from .fmsolve import (  # noqa: F401
    BatchSolveReport,
    InvalidArgument,
    MaskKind,
    MemoryCapExceeded,
    NormalEquations,
    RankDeficientError,
    RegularizedProblem,
    SingularSystemError,
    SolveReport,
    SolverOptions,
    build_mask,
    check_stationarity,
    make_problem,
    mask_commutativity,
    mask_resolvent,
    normal_equations,
    pipeline_device,
    project_to_spectral,
    solve_batched,
    solve_batched_many,
    solve_cuda,
    solve_cuda_many,
    solve_device,
    solve_host,
)

__all__ = [n for n in dir() if not n.startswith("_")]
