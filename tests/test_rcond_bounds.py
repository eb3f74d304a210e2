"""The rcond certificates chol_backsub_kernel uses before the exact Hager/Higham
estimator (csrc/fmap_tc.cu), checked in f64 on random SPD systems:

    ||A^{-1}||_1 <= max(M(L)^{-T} M(L)^{-1} e) <= max(M(L)^{-1} e) * max(M(L)^{-T} e)

for A = L L^T and M(L) the comparison matrix (|diag|, -|off-diagonal|).  Both are
upper bounds on ||A^{-1}||_1, so 1 / (||A||_1 * bound) never exceeds the true rcond
(the reference's estimate of ||A^{-1}||_1 never exceeds it either)."""
import numpy as np
import pytest


def _comparison(L):
    Mc = -np.abs(L)
    np.fill_diagonal(Mc, np.abs(np.diag(L)))
    return Mc


@pytest.mark.parametrize("k,seed,scale", [(8, 0, 1.0), (40, 1, 1e-3), (120, 2, 1e-6), (200, 3, 0.0)])
def test_certificate_bounds(k, seed, scale):
    rng = np.random.default_rng(seed)
    d = max(4, k // 2)
    A0 = rng.standard_normal((k, d))
    A = A0 @ A0.T + np.diag(scale + rng.uniform(0.0, 1.0, k) * 1e-2)  # rank-deficient Gram + small diagonal
    L = np.linalg.cholesky(A)
    Mc = _comparison(L)
    e = np.ones(k)
    u = np.linalg.solve(Mc, e)
    w = np.linalg.solve(Mc.T, e)
    w2 = np.linalg.solve(Mc.T, u)
    inv_norm = np.abs(np.linalg.inv(A)).sum(axis=0).max()
    rel = 1e-9 * max(1.0, inv_norm)
    assert inv_norm <= w2.max() * (1 + 1e-9) + rel
    assert w2.max() <= u.max() * w.max() * (1 + 1e-9) + rel
