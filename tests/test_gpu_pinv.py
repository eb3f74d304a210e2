"""GPU route for project_to_spectral (spectral.hpp:47-93): the reference's own
KATs (proj/tests/test_spectral.cpp:23-116) through fmap_project_pinv_f64, and
parity against the oracle's restatement (oracle.project_pinv) on random bases,
batched, in f64 and f32."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def randn(oracle, rows, cols, seed):
    return oracle.randn(rows, cols, seed)  # test_spectral.cpp:11-20


def test_kat_orthonormal_basis_is_exact(fm):  # test_spectral.cpp:23-28
    assert np.abs(fm.project_to_spectral(np.eye(3), np.eye(3)) - np.eye(3)).max() <= 1e-15


def test_kat_one_dimensional_least_squares(fm):  # :30-39
    a = fm.project_to_spectral(np.array([[2.0], [0.0]]), np.array([[4.0], [0.0]]))
    assert a.shape == (1, 1) and a[0, 0] == pytest.approx(2.0, rel=1e-14)


def test_kat_normal_equations(fm, oracle):  # :41-48
    B, F = randn(oracle, 20, 5, 101), randn(oracle, 20, 3, 102)
    expected = np.linalg.inv(B.T @ B) @ (B.T @ F)
    assert np.abs(fm.project_to_spectral(B, F) - expected).max() <= 1e-10


def test_kat_linear_in_features(fm, oracle):  # :50-58
    B, f1, f2 = randn(oracle, 15, 4, 7), randn(oracle, 15, 2, 8), randn(oracle, 15, 2, 9)
    lhs = fm.project_to_spectral(B, 0.37 * f1 - 1.85 * f2)
    rhs = 0.37 * fm.project_to_spectral(B, f1) - 1.85 * fm.project_to_spectral(B, f2)
    assert np.linalg.norm(lhs - rhs) <= 1e-12 * (1 + np.linalg.norm(rhs))


def test_kat_round_trip(fm, oracle):  # :60-67
    q, _ = np.linalg.qr(randn(oracle, 12, 5, 33))
    coeffs = randn(oracle, 5, 3, 34)
    assert np.abs(fm.project_to_spectral(q, q @ coeffs) - coeffs).max() <= 1e-12


def test_kat_rank_deficient(fm, oracle):  # :69-82
    B = np.zeros((4, 2))
    B[:, 0] = [1, 2, 3, 4]
    B[:, 1] = B[:, 0]
    with pytest.raises(fm.RankDeficientError) as ei:
        fm.project_to_spectral(B, randn(oracle, 4, 1, 55))
    assert ei.value.rank() == 1 and ei.value.expected() == 2


def test_kat_fewer_rows_than_columns(fm, oracle):  # :84-88
    with pytest.raises(fm.RankDeficientError):
        fm.project_to_spectral(randn(oracle, 2, 3, 56), randn(oracle, 2, 1, 57))


def test_kat_mismatched_dimensions(fm, oracle):  # :90-94
    with pytest.raises(fm.InvalidArgument):
        fm.project_to_spectral(randn(oracle, 6, 2, 58), randn(oracle, 5, 2, 59))


def test_kat_ill_conditioned_full_rank(fm):  # :96-106
    B = np.zeros((4, 2))
    B[0, 0], B[1, 1] = 1.0, 1e-12
    coeffs = np.array([[3.0], [5.0]])
    assert np.abs(fm.project_to_spectral(B, B @ coeffs) - coeffs).max() <= 1e-6


def test_kat_custom_condition_threshold(fm):  # :108-118
    B = np.zeros((4, 2))
    B[0, 0], B[1, 1] = 1.0, 1e-2
    coeffs = np.array([[-1.0], [2.0]])
    assert np.abs(fm.project_to_spectral(B, B @ coeffs, condition_threshold=10.0) - coeffs).max() <= 1e-10


def test_non_finite_rejected(fm, oracle):
    B = randn(oracle, 6, 2, 60)
    B[2, 1] = np.nan
    with pytest.raises(fm.InvalidArgument, match="basis"):
        fm.project_to_spectral(B, randn(oracle, 6, 1, 61))


@pytest.mark.parametrize("n,k,d", [(40, 6, 3), (300, 30, 12), (1200, 64, 32)])
def test_batched_parity_with_oracle(fm, oracle, n, k, d):
    b = 3
    B = np.stack([randn(oracle, n, k, 700 + q) for q in range(b)])
    F = np.stack([randn(oracle, n, d, 800 + q) for q in range(b)])
    got = fm.project_to_spectral(B, F)
    for q in range(b):
        ref = oracle.project_pinv(B[q], F[q])
        assert np.abs(got[q] - ref).max() <= 1e-9 * max(1.0, np.abs(ref).max())
    got32 = fm.project_to_spectral(B, F, precision="f32")
    assert np.abs(got32 - got).max() <= 1e-4 * max(1.0, np.abs(got).max())


def test_batch_names_lowest_rank_deficient_shape(fm, oracle):
    n, k = 30, 5
    B = np.stack([randn(oracle, n, k, 900 + q) for q in range(4)])
    B[2, :, 4] = B[2, :, 0] + B[2, :, 1]  # rank 4
    B[3, :, 3] = 0.0                      # rank 4
    F = np.stack([randn(oracle, n, 2, 950 + q) for q in range(4)])
    with pytest.raises(fm.RankDeficientError) as ei:
        fm.project_to_spectral(B, F)
    assert ei.value.rank() == 4 and "shape 2" in str(ei.value)


def test_mass_orthonormal_basis_agrees_with_the_hot_path_projection(fm, oracle):
    # for Phi^T M Phi = I the north_star projection Phi^T M F is the M-weighted
    # pinv; the Euclidean pinv of M^(1/2) Phi applied to M^(1/2) F is the same map
    from paper_2604_10377_b200 import synth
    phi, mass = synth.mass_orthonormal_basis(400, 12, 3, "1")
    F = randn(oracle, 400, 5, 77)
    s = np.sqrt(mass)[:, None]
    got = fm.project_to_spectral(s * phi, s * F)
    assert np.abs(got - phi.T @ (mass[:, None] * F)).max() <= 1e-10
