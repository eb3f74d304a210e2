"""Pin the CPU oracle (oracle/fmsolve_oracle.cpp) before trusting it.

The reference cannot be built here (Eigen/doctest/CLI11 absent)
and ships no golden solution vectors, so the oracle is pinned by
  * the reference's own known-answer tests and properties, restated from
    proj/tests/test_solver.cpp, test_masks.cpp, test_bench.cpp, acceptance.cpp;
  * the reference's golden memory table (tests/golden/memory_f32_k4_12.csv,
    copied by tests/golden/make_golden.py from proj/tests/golden/);
  * an independent LAPACK route (numpy.linalg / scipy) in float64.
CPU only; no GPU.
"""
import cmath
import csv
from pathlib import Path

import numpy as np
import pytest

GOLDEN = Path(__file__).resolve().parent / "golden"


def maxabs(x):
    return float(np.abs(x).max())


# ----------------------------------------------------------- solver KATs ----
def test_identity_descriptors(oracle):
    # test_solver.cpp:34-44
    k = 4
    eye = np.eye(k)
    G, R = oracle.normal_equations(eye, eye)
    M = np.zeros((k, k))
    for route in ("rowwise", "batched"):
        r = oracle.solve(G, R, M, 0.0, route=route)
        assert maxabs(r.maps - eye) <= 1e-14
        assert r.max_residual <= 1e-14
    assert maxabs(oracle.solve_full(G, R, M, 0.0) - eye) <= 1e-14


def test_oracle_k2(oracle):
    # test_solver.cpp:46-50
    eye = np.eye(2)
    G, R = oracle.normal_equations(eye, eye)
    assert maxabs(oracle.solve_full(G, R, np.zeros((2, 2)), 0.0) - eye) <= 1e-14


def test_closed_form_positive_mask(oracle):
    # test_solver.cpp:52-64
    k, lam = 8, 10.0
    eye = np.eye(k)
    mask = np.abs(oracle.randn(k, k, 21)) + 0.5
    G, R = oracle.normal_equations(eye, eye)
    C = oracle.solve(G, R, mask, lam, route="rowwise").maps
    expected = np.diag(1.0 / (1.0 + lam * np.diag(mask)))
    np.testing.assert_allclose(C, expected, rtol=1e-12, atol=1e-300)


def test_rowwise_vs_full_oracle(oracle):
    # test_solver.cpp:66-71
    G, R, M, _, _ = oracle.random_problem(16, 32, 77)
    assert maxabs(oracle.solve(G, R, M, 1.0, route="rowwise").maps - oracle.solve_full(G, R, M, 1.0)) <= 1e-8


def test_batched_vs_rowwise(oracle):
    # test_solver.cpp:73-78
    G, R, M, _, _ = oracle.random_problem(24, 48, 78)
    a = oracle.solve(G, R, M, 100.0, route="rowwise").maps
    b = oracle.solve(G, R, M, 100.0, route="batched").maps
    assert maxabs(a - b) <= 1e-10


@pytest.mark.parametrize("k", [4, 8, 16, 32])
def test_equivalence_triangle(oracle, k):
    # test_solver.cpp:80-97
    for lam in (0.0, 1.0, 100.0, 1e8):
        for seed in (11, 12):
            G, R, M, _, _ = oracle.random_problem(k, 2 * k, seed)
            rw = oracle.solve(G, R, M, lam, route="rowwise").maps
            bt = oracle.solve(G, R, M, lam, route="batched").maps
            full = oracle.solve_full(G, R, M, lam)
            assert maxabs(rw - bt) <= 1e-8
            assert maxabs(rw - full) <= 1e-8
            assert maxabs(bt - full) <= 1e-8


def test_stationarity_and_perturbation(oracle):
    # test_solver.cpp:99-114
    G, R, M, a, b = oracle.random_problem(12, 24, 90)
    lam = 100.0
    r = oracle.solve(G, R, M, lam, route="rowwise")
    bound = 1e-8 * (1.0 + np.linalg.norm(R))
    res = oracle.residual(r.maps, G, R, M, lam)
    assert res <= bound and r.max_residual <= bound
    pert = r.maps + 0.1 * oracle.randn(12, 12, 91)
    assert oracle.residual(pert, G, R, M, lam) > res


def test_unregularized_square_is_b_pinv_a(oracle):
    # test_solver.cpp:116-128
    k = 4
    a = oracle.randn(k, k, 92) + 4.0 * np.eye(k)
    b = oracle.randn(k, k, 93)
    M = np.zeros((k, k))
    expected = b @ np.linalg.pinv(a)
    G, R = oracle.normal_equations(a, b)
    assert oracle.residual(expected, G, R, M, 0.0) <= 1e-8
    assert maxabs(oracle.solve_full(G, R, M, 0.0) - expected) <= 1e-8
    assert maxabs(oracle.solve(G, R, M, 0.0, route="rowwise").maps - expected) <= 1e-8


def test_solution_is_energy_minimum(oracle):
    # test_solver.cpp:130-147
    k, d, lam = 8, 12, 1.0
    a, b, e1, e2 = oracle.generate_instance(k, d, 94)
    M = oracle.mask(0, e1, e2)
    G, R = oracle.normal_equations(a, b)
    C = oracle.solve(G, R, M, lam, route="rowwise").maps
    e0 = oracle.energy(C, a, b, M, lam)
    rng = np.random.default_rng(95)
    for _ in range(100):
        assert oracle.energy(C + 1e-3 * rng.standard_normal((k, k)), a, b, M, lam) > e0


def test_huge_lambda_kills_off_diagonal(oracle):
    # test_solver.cpp:149-162
    k = 8
    ev = np.arange(k, dtype=float)
    M = oracle.mask(0, ev, ev)
    a = oracle.randn(k, 2 * k, 96) / 4.0
    b = oracle.randn(k, 2 * k, 97) / 4.0
    G, R = oracle.normal_equations(a, b)
    C = oracle.solve(G, R, M, 1e8, route="rowwise").maps
    assert maxabs(C - np.diag(np.diag(C))) <= 1e-6


def test_stacked_batch_equals_individual(oracle):
    # test_solver.cpp:164-174
    probs = [oracle.random_problem(6, 12, 200 + q) for q in range(3)]
    G = np.stack([p[0] for p in probs])
    R = np.stack([p[1] for p in probs])
    M = np.stack([p[2] for p in probs])
    batch = oracle.solve(G, R, M, 100.0).maps
    for q in range(3):
        single = oracle.solve(G[q], R[q], M[q], 100.0, route="rowwise").maps
        assert maxabs(batch[q] - single) <= 1e-10


def test_underdetermined_is_singular(oracle):
    # test_solver.cpp:176-182
    G, R, M, _, _ = oracle.random_problem(8, 4, 98)
    for route in ("rowwise", "batched"):
        with pytest.raises(oracle.OracleError) as ei:
            oracle.solve(G, R, M, 0.0, route=route)
        assert ei.value.status == oracle.SINGULAR
    with pytest.raises(oracle.OracleError):
        oracle.solve_full(G, R, M, 0.0)


def test_singular_row_named_and_ridge(oracle):
    # test_solver.cpp:184-212
    a = np.zeros((3, 3))
    a[0, 0] = a[2, 2] = 1.0
    b = np.eye(3)
    M = np.zeros((3, 3))
    M[0, 1] = M[2, 1] = 1.0
    G, R = oracle.normal_equations(a, b)
    for route in ("rowwise", "batched"):
        with pytest.raises(oracle.OracleError) as ei:
            oracle.solve(G, R, M, 1.0, route=route)
        assert ei.value.failing_system == 1
        assert "1" in str(ei.value)
    oracle.solve(G, R, M, 1.0, route="rowwise", ridge=1e-3)


def test_memory_cap(oracle):
    # test_solver.cpp:214-225
    G, R, M, _, _ = oracle.random_problem(8, 16, 99)
    with pytest.raises(oracle.OracleError) as ei:
        oracle.solve(G, R, M, 1.0, memory_cap_bytes=10)
    assert ei.value.status == oracle.MEMORY_CAP
    assert ei.value.required_bytes == 8 * 8 * 8 * 8
    assert ei.value.cap_bytes == 10


def test_fault_injection(oracle):
    # test_solver.cpp:227-234
    G, R, M, _, _ = oracle.random_problem(10, 20, 100)
    a = oracle.solve(G, R, M, 100.0, route="rowwise").maps
    b = oracle.solve(G, R, M, 100.0, inject_fault=True).maps
    assert maxabs(a - b) > 1e-8


def test_thread_width_bitwise(oracle):
    # test_solver.cpp:236-244
    G, R, M, _, _ = oracle.random_problem(12, 24, 101)
    a = oracle.solve(G, R, M, 100.0, threads=1).maps
    b = oracle.solve(G, R, M, 100.0, threads=3).maps
    assert np.array_equal(a, b)


def test_peak_extra_bytes(oracle):
    # test_solver.cpp:246-251
    k = 10
    G, R, M, _, _ = oracle.random_problem(k, 2 * k, 102)
    assert oracle.solve(G, R, M, 1.0, route="rowwise").peak_extra_bytes == k * k * 8
    assert oracle.solve(G, R, M, 1.0).peak_extra_bytes == k * k * k * 8


def test_full_oracle_guard(oracle):
    # test_solver.cpp:253-259
    k = 65
    with pytest.raises(oracle.OracleError) as ei:
        oracle.solve_full(np.eye(k), np.eye(k), np.zeros((k, k)), 0.0)
    assert ei.value.status == oracle.INVALID_ARGUMENT


def test_input_validation(oracle):
    # test_solver.cpp:261-275
    G, R, M, _, _ = oracle.random_problem(4, 8, 105)
    with pytest.raises(oracle.OracleError):
        oracle.solve(G, R, M, -1.0)
    bad = M.copy()
    bad[1, 2] = -0.5
    with pytest.raises(oracle.OracleError):
        oracle.solve(G, R, bad, 1.0)
    nan = G.copy()
    nan[0, 0] = np.nan
    with pytest.raises(oracle.OracleError):
        oracle.solve(nan, R, M, 1.0)


def test_single_precision_mode(oracle):
    # test_solver.cpp:277-289
    a, b, e1, e2 = oracle.generate_instance(6, 12, 112)
    M = oracle.mask(0, e1, e2)
    G, R = oracle.normal_equations(a, b)
    G32, R32, M32 = (x.astype(np.float32) for x in (G, R, M))
    rw = oracle.solve(G32, R32, M32, 100.0, route="rowwise", dtype=np.float32).maps
    bt = oracle.solve(G32, R32, M32, 100.0, dtype=np.float32).maps
    full = oracle.solve_full(G32, R32, M32, 100.0, dtype=np.float32)
    assert maxabs(rw - bt) <= 1e-3 and maxabs(rw - full) <= 1e-3
    a, b, e1, e2 = oracle.generate_instance(8, 4, 113)
    M = oracle.mask(0, e1, e2).astype(np.float32)
    G, R = (x.astype(np.float32) for x in oracle.normal_equations(a, b))
    with pytest.raises(oracle.OracleError) as ei:
        oracle.solve(G, R, M, 0.0, route="rowwise", dtype=np.float32)
    assert ei.value.status == oracle.SINGULAR


def test_acceptance_exactness_sample(oracle):
    # acceptance.cpp:43-89 (every 10th instance, to keep the CPU suite short)
    tol = 1e-8
    worst_diff = worst_res = 0.0
    for k in (4, 8, 16, 32):
        for inst in range(0, 50, 10):
            seed = 1000 + 131 * k + inst
            G, R, M, a, b = oracle.random_problem(k, 2 * k, seed)
            scale = 1.0 + np.linalg.norm(R)
            for lam in (0.0, 1.0, 100.0):
                rw = oracle.solve(G, R, M, lam, route="rowwise")
                bt = oracle.solve(G, R, M, lam)
                full = oracle.solve_full(G, R, M, lam)
                worst_diff = max(worst_diff, maxabs(rw.maps - bt.maps), maxabs(rw.maps - full),
                                 maxabs(bt.maps - full))
                worst_res = max(worst_res, rw.max_residual / scale, bt.max_residual / scale,
                                oracle.residual(full, G, R, M, lam) / scale)
    assert worst_diff <= tol and worst_res <= tol


def test_lapack_cross_check(oracle):
    # independent route: numpy (LAPACK gesv) per row system, float64
    for k, d, seed, kind in ((20, 40, 3, 0), (50, 128, 4, 1), (64, 32, 5, 1)):
        G, R, M, _, _ = oracle.random_problem(k, d, seed, kind=kind)
        lam = 100.0
        C = oracle.solve(G, R, M, lam).maps
        ref = np.stack([np.linalg.solve(G + lam * np.diag(M[i]), R[i]) for i in range(k)])
        assert maxabs(C - ref) <= 1e-9 * max(1.0, maxabs(ref))


def test_rcond_estimate_matches_lapack_scale(oracle):
    # The Hager/Higham estimate must sit within the usual factor of the true
    # 1-norm rcond: an ill-conditioned but regular system passes at 1e-14 and
    # fails when the threshold is raised above its condition estimate.
    G, R, M, _, _ = oracle.random_problem(16, 32, 7)
    lam = 1.0
    S = G + lam * np.diag(M[0])
    true_rcond = 1.0 / (np.linalg.norm(S, 1) * np.linalg.norm(np.linalg.inv(S), 1))
    oracle.solve(G, R, M, lam, rcond_threshold=true_rcond / 10)
    with pytest.raises(oracle.OracleError):
        oracle.solve(G, R, M, lam, rcond_threshold=1.0)


# ------------------------------------------------------------- mask KATs ----
def test_commutativity_by_hand(oracle):
    # test_masks.cpp:10-19
    m = oracle.mask(0, [0, 1], [0, 2])
    assert m[0, 0] == 0 and m[0, 1] == 1 and m[1, 0] == 4 and m[1, 1] == 1


def test_commutativity_properties(oracle):
    # test_masks.cpp:21-41
    assert maxabs(np.diag(oracle.mask(0, [0, 1, 4], [0, 1, 4]))) == 0
    rng = np.random.default_rng(5)
    for _ in range(25):
        e1, e2 = np.sort(rng.uniform(0, 10, 6)), np.sort(rng.uniform(0, 10, 6))
        assert oracle.mask(0, e1, e2).min() >= 0
    with pytest.raises(oracle.OracleError):
        oracle.mask(0, [0, 1], [0, 1, 2])
    with pytest.raises(oracle.OracleError):
        oracle.mask(0, [-1, 0], [0, 1])


def test_resolvent_kats(oracle):
    # test_masks.cpp:53-100
    m = oracle.mask(1, [0, 0.5, 2, 7], [0, 0.5, 2, 7], 0.5)
    assert maxabs(np.diag(m)) == 0 and m.min() >= 0
    m = oracle.mask(1, [0, 1], [0, 1], 0.5)
    assert m[0, 1] > 0 and abs(m[0, 1] - m[1, 0]) <= 1e-14 * m[0, 1]
    rng = np.random.default_rng(17)
    sigma = 0.73
    e1, e2 = np.sort(rng.uniform(0, 5, 5)), np.sort(rng.uniform(0, 5, 5))
    m = oracle.mask(1, e1, e2, sigma)
    emax = max(e1.max(), e2.max())
    for i in range(5):
        for j in range(5):
            w2 = 1.0 / complex(e2[i] / emax, -sigma)
            w1 = 1.0 / complex(e1[j] / emax, -sigma)
            assert m[i, j] == pytest.approx(abs(w2 - w1) ** 2, rel=1e-12)
    for bad_sigma in (0.0, -1.0):
        with pytest.raises(oracle.OracleError):
            oracle.mask(1, [0, 1], [0, 1], bad_sigma)
    with pytest.raises(oracle.OracleError):
        oracle.mask(1, [0, 0], [0, 0], 0.5)


# ------------------------------------------------------- generator / golden --
def test_reference_generator(oracle):
    # test_bench.cpp:47-70
    a, b, e1, e2 = oracle.generate_instance(5, 10, 123)
    assert e1[0] == 0 and e2[0] == 0
    assert np.all(np.diff(e1) > 0) and np.all(np.diff(e2) > 0)
    a2, b2, e12, _ = oracle.generate_instance(5, 10, 123)
    assert np.array_equal(a, a2) and np.array_equal(b, b2) and np.array_equal(e1, e12)
    a3, _, _, _ = oracle.generate_instance(5, 10, 124)
    assert not np.array_equal(a, a3)
    G, R, M, _, _ = oracle.random_problem(16, 32, 7)
    oracle.solve(G, R, M, 0.0, route="rowwise")


def test_golden_memory_table(oracle):
    # proj/tests/golden/memory_f32_k4_12.csv: batched = b k^3 elem, loop = b k^2 elem
    rows = [r for r in csv.reader(open(GOLDEN / "memory_f32_k4_12.csv")) if r and not r[0].startswith("#")]
    header, body = rows[0], rows[1:]
    assert header == ["k", "precision", "batched_extra_bytes", "loop_working_set_bytes", "ratio"]
    for k_s, prec, batched, loop, ratio in body:
        k = int(k_s)
        G, R, M, _, _ = oracle.random_problem(k, 2 * k, 42)
        G, R, M = (x.astype(np.float32) for x in (G, R, M))
        assert oracle.solve(G, R, M, 100.0, dtype=np.float32).peak_extra_bytes == int(batched)
        assert oracle.solve(G, R, M, 100.0, route="rowwise", dtype=np.float32).peak_extra_bytes == int(loop)
        assert int(ratio) == k and prec == "f32"


def test_acceptance_memory_claim(oracle):
    # acceptance.cpp:170-199: k=300, b=1 -> 108,000,000 B (f32), 216,000,000 B (f64)
    assert 300 ** 3 * 4 == 108_000_000 and 300 ** 3 * 8 == 216_000_000


def test_projection_restatement(oracle):
    # north_star stage (1): Phi^T diag(Mass) F, vs numpy in float64
    rng = np.random.default_rng(3)
    phi, mass, F = rng.standard_normal((50, 7)), rng.uniform(0.5, 1.5, 50) / 50, rng.standard_normal((50, 5))
    np.testing.assert_allclose(oracle.project_mass(phi, mass, F), phi.T @ (mass[:, None] * F), rtol=1e-12, atol=1e-14)


def test_golden_solutions_fixture(oracle):
    # tests/golden/solutions.npz (tests/golden/make_golden.py): the oracle must
    # keep reproducing its committed float64 solutions.
    z = np.load(GOLDEN / "solutions.npz")
    for name in sorted({n.split("__")[0] for n in z.files}):
        G, R, M, lam, C = (z[f"{name}__{s}"] for s in ("G", "R", "M", "lam", "C"))
        out = oracle.solve(G, R, M, float(lam)).maps
        assert maxabs(out - C) <= 1e-12 * max(1.0, maxabs(C))


def test_generator_golden(oracle):
    # pins the libstdc++ engine/distribution stream the reference generator uses
    z = np.load(GOLDEN / "generator.npz")
    a, b, e1, e2 = oracle.generate_instance(5, 10, 123)
    assert np.array_equal(a, z["a"]) and np.array_equal(b, z["b"])
    assert np.array_equal(e1, z["ev1"]) and np.array_equal(e2, z["ev2"])
