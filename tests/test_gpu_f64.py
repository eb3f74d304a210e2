"""GPU parity of the f64 route (fmap_solve_f64, csrc/fmap_f64.cu) against the CPU
oracle's f64 batched route — the reference's default precision (bench.hpp:32)
and verify tolerance 1e-8 (bench.cpp:28), rcond threshold 1e-14
(solver.hpp:18-27).  KATs follow proj/tests/test_solver.cpp (cited per test)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-8  # bench.cpp:28 verify tolerance for f64 (absolute, on the maps)


def _problems(oracle, b, k, d, seed, kind=1):
    Gs, Rs, Ms = [], [], []
    for q in range(b):
        G, R, M, _, _ = oracle.random_problem(k, d, seed + q, kind=kind)
        Gs.append(G)
        Rs.append(R)
        Ms.append(M)
    return np.stack(Gs), np.stack(Rs), np.stack(Ms)


@pytest.mark.parametrize("k,b", [(1, 3), (5, 3), (16, 3), (40, 3), (100, 2), (200, 1), (234, 1), (240, 2),
                                 (300, 2)])
def test_f64_route_matches_reference_batched_f64(fm, oracle, k, b):
    G, R, M = _problems(oracle, b, k, 2 * k if k < 128 else 256, 500 + k, kind=0 if k == 1 else 1)
    lam = 100.0
    out = fm.solve_host(G, R, M, lam, precision="f64")
    assert out.maps.dtype == np.float64
    ref = oracle.solve(G, R, M, lam, route="batched", dtype=np.float64, threads=0)
    assert np.abs(out.maps - ref.maps).max() <= TOL
    # the reported residual is the reference's ||C G + lam M.*C - R||_F (max over pairs)
    assert out.max_residual_norm == pytest.approx(ref.max_residual, rel=1e-3, abs=1e-12)


def test_f64_identity_and_closed_form(fm, oracle):
    # test_solver.cpp:34-64: A = B = I -> C = diag(1 / (1 + lambda M_ii))
    k = 6
    eye = np.eye(k)
    M = np.abs(oracle.randn(k, k, 3))
    out = fm.solve_host(eye[None], eye[None], M[None], 2.5, precision="f64").maps[0]
    assert np.abs(out - np.diag(1.0 / (1.0 + 2.5 * np.diag(M)))).max() <= 1e-14


def test_f64_singular_lowest_index(fm, oracle):
    # test_solver.cpp:187-203: a singular pair names its first row system
    G, R, M = _problems(oracle, 3, 12, 24, 40, kind=0)
    G[1] = 0.0
    M[1] = 0.0
    with pytest.raises(fm.SingularSystemError) as ei:
        fm.solve_host(G, R, M, 100.0, precision="f64")
    assert ei.value.system() == 12


def test_f64_validation_and_limits(fm, oracle):
    G, R, M = _problems(oracle, 2, 8, 16, 41)
    bad = M.copy()
    bad[0, 1, 2] = -1.0
    with pytest.raises(fm.InvalidArgument, match="non-negative"):
        fm.solve_host(G, R, bad, 1.0, precision="f64")
    nan = R.copy()
    nan[1, 0, 0] = np.nan
    with pytest.raises(fm.InvalidArgument, match="rhs"):
        fm.solve_host(G, nan, M, 1.0, precision="f64")
    with pytest.raises(fm.InvalidArgument):
        fm.solve_host(G, R, M, -1.0, precision="f64")
    k = 513  # beyond the f64 route's limit (rows past shared memory spill to L2 up to k = 512)
    z = np.zeros((1, k, k))
    with pytest.raises(fm.InvalidArgument, match="f64 route"):
        fm.solve_host(z + np.eye(k), z, z, 1.0, precision="f64")
    with pytest.raises(fm.MemoryCapExceeded):
        fm.solve_host(G, R, M, 1.0, fm.SolverOptions(memory_cap_bytes=10), precision="f64")


def test_f64_fault_hook_matches_reference_fault(fm, oracle):
    # solver.hpp:269-273 via test_solver.cpp:277-292: the injected fault changes
    # pair 0 row 0 exactly as the reference's faulted batched solve does
    G, R, M = _problems(oracle, 2, 20, 40, 42)
    clean = fm.solve_host(G, R, M, 100.0, precision="f64").maps
    faulted = fm.solve_host(G, R, M, 100.0, fm.SolverOptions(inject_fault=True), precision="f64").maps
    ref = oracle.solve(G, R, M, 100.0, route="batched", dtype=np.float64, threads=0, inject_fault=True).maps
    assert np.abs(faulted - clean).max() > 1e-6
    assert np.abs(faulted - ref).max() <= 1e-9 * max(1.0, np.abs(ref).max())


@pytest.mark.parametrize("k", [24, 240])
def test_f64_rcond_verdict_matches_reference(fm, oracle, k):
    # solver.hpp:164-168 in f64 (threshold 1e-14 by default): thresholds placed on
    # both sides of the reference's estimate force the exact Hager/Higham path;
    # the verdict and the estimate must agree (k = 240 runs the spilled kernel)
    rng = np.random.default_rng(k)
    Q, _ = np.linalg.qr(rng.standard_normal((k, k)))
    G = (Q * np.logspace(0, -6, k)) @ Q.T
    G = 0.5 * (G + G.T)
    R = rng.standard_normal((k, k))
    M = np.zeros((k, k))
    r0 = oracle.rcond(G, np.float64)
    ok = fm.solve_host(G[None], R[None], M[None], 0.0, fm.SolverOptions(rcond_threshold=r0 / 1.5), precision="f64")
    assert 0.95 <= ok.min_rcond / r0 <= 1.05
    assert ok.rcond_exact_systems == k
    with pytest.raises(fm.SingularSystemError) as ei:
        fm.solve_host(G[None], R[None], M[None], 0.0, fm.SolverOptions(rcond_threshold=r0 * 1.5), precision="f64")
    assert ei.value.system() == 0
    # the default threshold (1e-14) accepts it
    out = fm.solve_host(G[None], R[None], M[None], 0.0, precision="f64")
    assert out.min_rcond >= 1e-14
