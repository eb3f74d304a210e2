"""GPU singular verdict vs the reference's rcond test (solver.hpp:158-168).

The reference rejects a row system when PartialPivLU::rcond() -- a Hager/Higham
estimate of 1 / (||A||_1 ||A^{-1}||_1) -- is below the threshold (1e-7 for f32).
The GPU route proves acceptance with a comparison-matrix certificate and, when
that is inconclusive, runs the same Hager/Higham estimator on its Cholesky
factor.  These tests build SPD systems with a controlled spectrum, read the
reference's estimate from the oracle (oracle.rcond: LU + Hager/Higham, the
restatement of solver.hpp:158-166) and require the GPU verdict to agree on both
sides of thresholds placed around it -- which forces the exact-estimator path.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _spd(k, cond, seed, rot=True):
    rng = np.random.default_rng(seed)
    ev = np.logspace(0.0, -np.log10(cond), k)
    if not rot:
        return np.diag(ev)
    Q, _ = np.linalg.qr(rng.standard_normal((k, k)))
    G = (Q * ev) @ Q.T
    return 0.5 * (G + G.T)


def _system(k, cond, seed):
    G = _spd(k, cond, seed).astype(np.float32)
    R = np.random.default_rng(seed + 1).standard_normal((k, k)).astype(np.float32)
    M = np.zeros((k, k), np.float32)  # A_i = G for every row i
    return G, R, M


@pytest.mark.parametrize("k,cond,seed", [(24, 1e3, 1), (50, 2e4, 2), (96, 5e3, 3), (200, 1e4, 4)])
def test_verdict_matches_reference_estimate_around_threshold(fm, oracle, k, cond, seed):
    G, R, M = _system(k, cond, seed)
    r0 = oracle.rcond(G, np.float32)
    assert r0 > 0
    # accept side: threshold below the estimate but above half the certificate
    # bound, so the exact estimator decides
    ok = fm.solve_host(G[None], R[None], M[None], 0.0, fm.SolverOptions(rcond_threshold=r0 / 1.5))
    assert 0.9 <= ok.min_rcond / r0 <= 1.1, (ok.min_rcond, r0)
    ref = oracle.solve(G, R, M, 0.0, dtype=np.float32, rcond_threshold=r0 / 1.5).maps
    scale = np.abs(ref).max()
    # both are fp32 factorizations of a system with cond ~ `cond` (no lambda term)
    assert np.abs(ok.maps[0] - ref).max() <= max(1e-4, 5e-8 * cond) * scale
    # reject side: the reference raises, so must the GPU (lowest system = 0)
    with pytest.raises(oracle.OracleError):
        oracle.solve(G, R, M, 0.0, dtype=np.float32, rcond_threshold=r0 * 1.5)
    with pytest.raises(fm.SingularSystemError) as ei:
        fm.solve_host(G[None], R[None], M[None], 0.0, fm.SolverOptions(rcond_threshold=r0 * 1.5))
    assert ei.value.system() == 0


def test_default_threshold_both_sides(fm, oracle):
    # 1e-7 (solver.hpp:25): a well-conditioned system passes (certificate path), a
    # system with rcond ~1e-9 fails on both routes.
    k = 32
    G, R, M = _system(k, 1e2, 7)
    assert oracle.rcond(G, np.float32) > 1e-3
    out = fm.solve_host(G[None], R[None], M[None], 0.0)
    assert out.min_rcond > 1e-7
    Gb = _spd(k, 1e9, 8, rot=False).astype(np.float32)  # diagonal: exact pivots, rcond = 1e-9
    r0 = oracle.rcond(Gb, np.float32)
    assert 0 < r0 < 1e-7
    with pytest.raises(fm.SingularSystemError):
        fm.solve_host(Gb[None], R[None], M[None], 0.0)


def test_mixed_batch_lowest_failing_system(fm, oracle):
    # pair 0 well conditioned, pair 1's every row below a threshold between the
    # two estimates: the failing index is the first system of pair 1.
    k = 40
    G0, R0, M0 = _system(k, 1e2, 11)
    G1, R1, M1 = _system(k, 3e4, 12)
    r1 = oracle.rcond(G1, np.float32)
    thr = r1 * 2.0
    assert oracle.rcond(G0, np.float32) > 4 * thr
    G, R, M = np.stack([G0, G1]), np.stack([R0, R1]), np.stack([M0, M1])
    with pytest.raises(fm.SingularSystemError) as ei:
        fm.solve_host(G, R, M, 0.0, fm.SolverOptions(rcond_threshold=thr))
    assert ei.value.system() == k


def test_certificate_never_rejects_baseline_systems(fm, oracle):
    # BASELINE-like resolvent systems (rcond ~1e-5..1e-4 >> 1e-7): accepted, and
    # the reported rcond is a lower bound of the reference's estimate.
    G, R, M, _, _ = oracle.random_problem(60, 128, 21, kind=1)
    lam = 100.0
    out = fm.solve_host(G[None].astype(np.float32), R[None].astype(np.float32), M[None].astype(np.float32), lam)
    worst = min(oracle.rcond((G + lam * np.diag(M[i])).astype(np.float32), np.float32) for i in range(60))
    assert 1e-7 < out.min_rcond <= worst * 1.05
