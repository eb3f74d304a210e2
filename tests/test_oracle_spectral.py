"""The oracle's project_to_spectral restatement (oracle/fmsolve_oracle.cpp,
spectral.hpp:47-93) pinned by the reference's own KATs
(proj/tests/test_spectral.cpp:23-116) and by numpy's pinv — CPU only."""
import numpy as np
import pytest

import oracle


def randn(rows, cols, seed):
    return oracle.randn(rows, cols, seed)  # test_spectral.cpp:11-20 (mt19937_64 + normal)


def test_orthonormal_basis_is_exact():  # test_spectral.cpp:23-28
    a = oracle.project_pinv(np.eye(3), np.eye(3))
    assert np.abs(a - np.eye(3)).max() <= 1e-15


def test_one_dimensional_least_squares():  # :30-39
    a = oracle.project_pinv(np.array([[2.0], [0.0]]), np.array([[4.0], [0.0]]))
    assert a.shape == (1, 1) and a[0, 0] == pytest.approx(2.0, rel=1e-14)


def test_matches_explicit_normal_equations():  # :41-48
    B, F = randn(20, 5, 101), randn(20, 3, 102)
    expected = np.linalg.inv(B.T @ B) @ (B.T @ F)
    assert np.abs(oracle.project_pinv(B, F) - expected).max() <= 1e-10


def test_linear_in_features():  # :50-58
    B, f1, f2 = randn(15, 4, 7), randn(15, 2, 8), randn(15, 2, 9)
    lhs = oracle.project_pinv(B, 0.37 * f1 - 1.85 * f2)
    rhs = 0.37 * oracle.project_pinv(B, f1) - 1.85 * oracle.project_pinv(B, f2)
    assert np.linalg.norm(lhs - rhs) <= 1e-12 * (1 + np.linalg.norm(rhs))


def test_round_trip_orthonormal_basis():  # :60-67
    q, _ = np.linalg.qr(randn(12, 5, 33))
    coeffs = randn(5, 3, 34)
    assert np.abs(oracle.project_pinv(q, q @ coeffs) - coeffs).max() <= 1e-12


def test_rank_deficient_reports_rank():  # :69-82
    B = np.zeros((4, 2))
    B[:, 0] = [1, 2, 3, 4]
    B[:, 1] = B[:, 0]
    with pytest.raises(oracle.OracleError) as ei:
        oracle.project_pinv(B, randn(4, 1, 55))
    assert ei.value.status == oracle.RANK_DEFICIENT and ei.value.rank == 1 and ei.value.expected == 2


def test_fewer_rows_than_columns():  # :84-88
    with pytest.raises(oracle.OracleError) as ei:
        oracle.project_pinv(randn(2, 3, 56), randn(2, 1, 57))
    assert ei.value.status == oracle.RANK_DEFICIENT


def test_ill_conditioned_full_rank_fallback():  # :96-106
    B = np.zeros((4, 2))
    B[0, 0], B[1, 1] = 1.0, 1e-12
    coeffs = np.array([[3.0], [5.0]])
    assert np.abs(oracle.project_pinv(B, B @ coeffs) - coeffs).max() <= 1e-6


def test_custom_condition_threshold():  # :108-118
    B = np.zeros((4, 2))
    B[0, 0], B[1, 1] = 1.0, 1e-2
    coeffs = np.array([[-1.0], [2.0]])
    assert np.abs(oracle.project_pinv(B, B @ coeffs, condition_threshold=10.0) - coeffs).max() <= 1e-10


@pytest.mark.parametrize("n,k,d", [(50, 7, 3), (300, 40, 16)])
def test_matches_numpy_pinv(n, k, d):
    B, F = randn(n, k, 200 + k), randn(n, d, 300 + k)
    assert np.abs(oracle.project_pinv(B, F) - np.linalg.pinv(B) @ F).max() <= 1e-9
