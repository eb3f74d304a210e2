"""GPU parity: libfmap_cuda's solver vs the CPU oracle (restated reference
solver, oracle/fmsolve_oracle.cpp) on identical seeded inputs.

Bar (BASELINE.json north_star): max|dC| <= 1e-4 * ||C||_max against the
reference f32 route, relative residual <= 1e-5.  Restated KATs follow
proj/tests/test_solver.cpp (file:line cited per test).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL_REL = 1e-4   # north_star: max|dC| <= 1e-4 * ||C||_max
RES_REL = 1e-5   # north_star: relative residual <= 1e-5 (fp32)


def _ref(oracle, G, R, M, lam, **kw):
    return oracle.solve(G, R, M, lam, route="batched", dtype=np.float32, threads=0, **kw).maps


def _ref64(oracle, G, R, M, lam, **kw):
    return oracle.solve(G, R, M, lam, route="batched", dtype=np.float64, threads=0, **kw).maps


def _assert_parity(C, Cref, what=""):
    scale = np.abs(Cref).max()
    err = np.abs(C.astype(np.float64) - Cref.astype(np.float64)).max()
    assert err <= TOL_REL * scale, f"{what}: max|dC|={err:.3e} > {TOL_REL}*{scale:.3e}"


def _rel_residual(oracle, C, G, R, M, lam):
    worst = 0.0
    for q in range(G.shape[0]):
        r = oracle.residual(C[q], G[q], R[q], M[q], lam)
        worst = max(worst, r / np.linalg.norm(R[q].astype(np.float64)))
    return worst


def _problems(oracle, b, k, d, seed, kind=1, sigma=0.5):
    Gs, Rs, Ms = [], [], []
    for q in range(b):
        G, R, M, _, _ = oracle.random_problem(k, d, seed + q, kind=kind, sigma=sigma)
        Gs.append(G)
        Rs.append(R)
        Ms.append(M)
    return (np.stack(Gs).astype(np.float32), np.stack(Rs).astype(np.float32),
            np.stack(Ms).astype(np.float32))


def test_identity_descriptors_give_identity(fm, oracle):
    # test_solver.cpp:34-44
    k = 4
    eye = np.eye(k)
    rep = fm.solve_cuda(eye, eye, np.zeros((k, k)), 0.0)
    assert np.abs(rep.map - eye).max() <= 1e-6
    assert rep.residual_norm <= 1e-6


def test_closed_form_diagonal(fm, oracle):
    # test_solver.cpp:52-64: A=B=I, M>0 -> C = diag(1/(1+lambda M_ii))
    k, lam = 8, 10.0
    mask = np.abs(oracle.randn(k, k, 21)) + 0.5
    eye = np.eye(k)
    rep = fm.solve_cuda(eye, eye, mask, lam)
    expected = np.diag(1.0 / (1.0 + lam * np.diag(mask)))
    assert np.abs(rep.map - expected).max() <= 1e-6 * np.abs(expected).max() * 10


@pytest.mark.parametrize("k", [1, 2, 3, 5, 8, 16, 17, 24, 32, 50])
def test_small_k_vs_oracle_and_full(fm, oracle, k):
    # test_solver.cpp:66-71 / :80-97 (triangle) at fp32
    d = 2 * k
    G, R, M = _problems(oracle, 3, k, d, 77, kind=0)
    for lam in (1.0, 100.0):
        C = fm.solve_host(G, R, M, lam).maps
        _assert_parity(C, _ref(oracle, G, R, M, lam), f"k={k} lam={lam}")
        if k <= 16:
            full = oracle.solve_full(G[0], R[0], M[0], lam)
            _assert_parity(C[0], full, f"full k={k}")


@pytest.mark.parametrize("k", list(range(20, 301, 20)))
def test_k_sweep_cfg3_shapes(fm, oracle, k):
    # BASELINE cfg3 resolutions (d=256); 2 pairs vs the f32 reference route,
    # relative residual on all of them.
    G, R, M = _problems(oracle, 2, k, 256, 1000 + k, kind=1)
    lam = 100.0
    out = fm.solve_host(G, R, M, lam)
    _assert_parity(out.maps, _ref(oracle, G, R, M, lam), f"k={k}")
    assert _rel_residual(oracle, out.maps, G, R, M, lam) <= RES_REL


def test_headline_shape_subset(fm, oracle):
    # cfg2 shape (k=200, d=256): 64 pairs on the GPU, 4 checked against the oracle
    G, R, M = _problems(oracle, 64, 200, 256, 5)
    lam = 100.0
    out = fm.solve_host(G, R, M, lam)
    sub = slice(0, 4)
    _assert_parity(out.maps[sub], _ref(oracle, G[sub], R[sub], M[sub], lam), "cfg2 subset")
    assert out.max_residual_norm / max(np.linalg.norm(R[q]) for q in range(64)) <= RES_REL * 10
    assert _rel_residual(oracle, out.maps[:8], G[:8], R[:8], M[:8], lam) <= RES_REL


def test_singular_detected_and_named(fm, oracle):
    # test_solver.cpp:184-212: gram = diag(1,0,1); mask row 1 all zero -> system 1 singular
    a = np.zeros((3, 3))
    a[0, 0] = a[2, 2] = 1.0
    b = np.eye(3)
    mask = np.zeros((3, 3))
    mask[0, 1] = mask[2, 1] = 1.0
    with pytest.raises(fm.SingularSystemError) as ei:
        fm.solve_cuda(a, b, mask, 1.0)
    assert ei.value.system() == 1
    assert "1" in str(ei.value)
    fm.solve_cuda(a, b, mask, 1.0, fm.SolverOptions(ridge=1e-3))


def test_underdetermined_unregularized_is_singular(fm, oracle):
    # test_solver.cpp:176-182 and :286-288 (f32 thin instance)
    G, R, M, _, _ = oracle.random_problem(8, 4, 98)
    with pytest.raises(fm.SingularSystemError):
        fm.solve_host(G[None], R[None], M[None], 0.0)


def test_lowest_failing_index_wins(fm, oracle):
    G, R, M = _problems(oracle, 4, 6, 12, 200, kind=0)
    G[2] = 0.0  # pair 2 singular at lambda=0 (every row)
    G[3] = 0.0
    with pytest.raises(fm.SingularSystemError) as ei:
        fm.solve_host(G, R, M, 0.0)
    assert ei.value.system() == 2 * 6


def test_input_validation(fm, oracle):
    # test_solver.cpp:261-275
    G, R, M, a, b = oracle.random_problem(4, 8, 105)
    with pytest.raises(fm.InvalidArgument):
        fm.solve_host(G[None], R[None], M[None], -1.0)
    bad = M.copy()
    bad[1, 2] = -0.5
    with pytest.raises(fm.InvalidArgument):
        fm.solve_host(G[None], R[None], bad[None], 1.0)
    nan = G.copy()
    nan[0, 0] = np.nan
    with pytest.raises(fm.InvalidArgument):
        fm.solve_host(nan[None], R[None], M[None], 1.0)
    with pytest.raises(fm.InvalidArgument):
        fm.solve_cuda(oracle.randn(4, 8, 108), oracle.randn(5, 8, 109), np.zeros((4, 4)), 1.0)


def test_memory_cap(fm, oracle):
    # test_solver.cpp:214-225 (cuda-route accounting)
    G, R, M, _, _ = oracle.random_problem(8, 16, 99)
    with pytest.raises(fm.MemoryCapExceeded) as ei:
        fm.solve_host(G[None], R[None], M[None], 1.0, fm.SolverOptions(memory_cap_bytes=10))
    assert ei.value.cap_bytes() == 10
    assert ei.value.required_bytes() > 10


def test_fault_injection_diverges_and_matches_reference_fault(fm, oracle):
    # test_solver.cpp:227-234; the faulted system is solved exactly, so it also
    # matches the reference's faulted batched route.
    G, R, M, _, _ = oracle.random_problem(10, 20, 100)
    lam = 100.0
    clean = fm.solve_host(G[None], R[None], M[None], lam).maps
    faulted = fm.solve_host(G[None], R[None], M[None], lam, fm.SolverOptions(inject_fault=True)).maps
    assert np.abs(clean - faulted).max() > 1e-3
    ref = _ref64(oracle, G[None], R[None], M[None], lam, inject_fault=True)
    _assert_parity(faulted, ref, "fault")


def test_deterministic(fm, oracle):
    # test_solver.cpp:236-244 analogue: bitwise identical across calls
    G, R, M = _problems(oracle, 8, 40, 80, 101)
    a = fm.solve_host(G, R, M, 100.0).maps
    b = fm.solve_host(G, R, M, 100.0).maps
    assert np.array_equal(a, b)


def test_stacked_batch_equals_individual(fm, oracle):
    # test_solver.cpp:164-174
    G, R, M = _problems(oracle, 3, 6, 12, 200, kind=0)
    batch = fm.solve_host(G, R, M, 100.0).maps
    for q in range(3):
        single = fm.solve_host(G[q:q + 1], R[q:q + 1], M[q:q + 1], 100.0).maps[0]
        assert np.array_equal(batch[q], single)


@pytest.mark.parametrize("env", [{}, {"FMAP_TC_NS": "2"}, {"FMAP_TC_NOTMA": "1"},
                                 {"FMAP_TC_NS": "2", "FMAP_TC_NOTMA": "1"}],
                         ids=["tma", "ns2-tma", "ldg", "ns2-ldg"])
@pytest.mark.parametrize("k,b", [(200, 4), (40, 24), (64, 12), (36, 40)])
def test_tensor_core_staging_variants(fm, oracle, monkeypatch, env, k, b):
    # Enough systems for several per CTA (148 SMs x 2), so the next system's G is
    # staged during the current one's panels (TMA + tcgen05.cp) — and the per-thread
    # load path and the two-systems-per-CTA layout give the same answers.
    for key, v in env.items():
        monkeypatch.setenv(key, v)
    G, R, M = _problems(oracle, b, k, 96, 300 + k)
    lam = 100.0
    out = fm.solve_host(G, R, M, lam)
    sub = slice(0, 2)
    _assert_parity(out.maps[sub], _ref(oracle, G[sub], R[sub], M[sub], lam), f"k={k} {env}")
    assert _rel_residual(oracle, out.maps, G, R, M, lam) <= RES_REL
    monkeypatch.delenv("FMAP_TC_NS", raising=False)
    monkeypatch.delenv("FMAP_TC_NOTMA", raising=False)
    base = fm.solve_host(G, R, M, lam).maps
    assert np.array_equal(out.maps, base) or env.get("FMAP_TC_NS") == "2"


def test_host_copy_pipeline_matches_unpipelined(fm, oracle, monkeypatch):
    # The host entry overlaps chunked H2D / solve / D2H (default 4 chunks for >= 8
    # pairs; G and M land before R, the factorization starts before R and before
    # validation) and computes the residual once every chunk is solved (tcgen05);
    # 37 pairs make the last chunk partial.  The maps are bitwise the unpipelined ones, the
    # reported residual agrees, and parity holds on the tail chunk.
    G, R, M = _problems(oracle, 37, 40, 64, 77)
    for res in (True, False):
        opts = fm.SolverOptions(compute_residual=res)
        piped = fm.solve_host(G, R, M, 100.0, opts)
        launches = fm._lib.context(0).last_launches
        assert launches.count("chol_tc_kernel") > 1 and ("gram_tc_kernel(residual)" in launches) == res, launches
        monkeypatch.setenv("FMAP_PIPELINE", "1")
        plain = fm.solve_host(G, R, M, 100.0, opts)
        monkeypatch.delenv("FMAP_PIPELINE")
        assert np.array_equal(piped.maps, plain.maps)
        if res:
            # both are fp32 evaluations of a ~zero residual (different summation
            # orders): compare at the north_star bar, not bitwise
            rmax = max(np.linalg.norm(R[q].astype(np.float64)) for q in range(G.shape[0]))
            assert 0 < piped.max_residual_norm <= RES_REL * rmax
            assert 0 < plain.max_residual_norm <= RES_REL * rmax
    _assert_parity(piped.maps[-3:], _ref(oracle, G[-3:], R[-3:], M[-3:], 100.0), "pipelined tail chunk")


@pytest.mark.parametrize("what", ["nan", "nan_gram_first_chunk", "negative_mask", "singular"])
def test_host_copy_pipeline_error_exposes_no_partial_result(fm, oracle, what):
    # An error found in the LAST chunk (after earlier chunks were already copied
    # back) must not leave partial maps in the caller's buffer.
    import ctypes as C
    from paper_2604_10377_b200 import _lib, fmsolve
    G, R, M = _problems(oracle, 32, 24, 48, 91)
    if what == "nan":  # in R: found by the validation that runs after the factorization
        R[31, 5, 7] = np.nan
        expect = fm.InvalidArgument
    elif what == "nan_gram_first_chunk":  # the factorization sees it first; INVALID_ARGUMENT still wins
        G[0, 3, 3] = np.nan
        expect = fm.InvalidArgument
    elif what == "negative_mask":
        M[20, 2, 9] = -1.0
        expect = fm.InvalidArgument
    else:
        G[31] = 0.0
        M[31] = 0.0
        expect = fm.SingularSystemError
    out = np.full(G.shape, 7.0, np.float32)
    ctx = fmsolve._ctx(0)
    o = fmsolve.SolverOptions().to_c()
    rep = _lib.ReportC()
    P = lambda x: C.c_void_p(x.ctypes.data)  # noqa: E731
    st = ctx._lib.fmap_solve_f32(ctx.handle, 32, 24, P(G), P(R), P(M), C.c_float(100.0), C.byref(o), P(out),
                                 C.byref(rep))
    assert st != 0
    with pytest.raises(expect):
        fmsolve._raise(ctx, st, rep)
    assert "chol_tc_kernel" in ctx.last_launches and ctx.last_launches.count("chol_tc_kernel") > 1  # pipelined
    assert np.all(out == 0.0)  # earlier chunks were copied back: zero-filled, no partial result


@pytest.mark.timeout(240, method="thread")
def test_repeated_cfg2_solves_terminate_and_repeat_bitwise(fm):
    # Hundreds of back-to-back cfg2-sized solves through the device entry, the fused
    # eigenvalue-mask entry and the copy-pipelined host entry (residual on), as the
    # bench runs them: the mbarrier protocol of the solver must never deadlock (a
    # phase race between finished row groups and the MMA warp once hung about one
    # host solve in fifty), and every repetition returns the same maps.
    import torch
    from paper_2604_10377_b200 import synth
    G, R, e1, e2 = synth.random_normal_equations(64, 200, 256, 7)
    M = fm.build_mask(fm.MaskKind.Resolvent, e1, e2, 0.5)
    dev = torch.device("cuda", 0)
    tG, tR, tM, t1, t2 = (torch.from_numpy(x).to(dev) for x in (G, R, M, e1, e2))
    opts = fm.SolverOptions(compute_residual=False)
    base, _ = fm.solve_device(tG, tR, tM, lam=100.0, opts=opts)
    for _ in range(100):
        C, _ = fm.solve_device(tG, tR, tM, lam=100.0, opts=opts)
        assert torch.equal(C, base)
    for _ in range(50):
        fm.solve_device(tG, tR, lam=100.0, ev1=t1, ev2=t2, opts=opts)
    host = fm.solve_host(G, R, M, 100.0).maps
    for _ in range(100):
        assert np.array_equal(fm.solve_host(G, R, M, 100.0).maps, host)


@pytest.mark.parametrize("k,b", [(80, 24), (100, 24), (128, 20), (144, 16)])
def test_register_capped_residency_variants(fm, oracle, k, b):
    # k = 65..144 run 96-register builds of the solver so the register file holds as
    # many CTAs per SM as tensor memory allows (5 / 4 / 3 instead of 4 / 3 / 2), on a
    # persistent grid of exactly the resident CTAs; enough systems here for several
    # per CTA, so the next system's staging path runs as well.
    G, R, M = _problems(oracle, b, k, 128, 4000 + k)
    lam = 100.0
    out = fm.solve_host(G, R, M, lam)
    sub = slice(0, 2)
    _assert_parity(out.maps[sub], _ref(oracle, G[sub], R[sub], M[sub], lam), f"k={k}")
    assert _rel_residual(oracle, out.maps, G, R, M, lam) <= RES_REL


def test_report_factor_seconds(fm, oracle):
    # fmap_report.factor_seconds: CUDA events around the factorization launch alone
    # (bench.py's roofline on the dominant kernel), inside wall_seconds (whole solve)
    import torch
    G, R, M = _problems(oracle, 4, 120, 96, 77)
    dev = torch.device("cuda", 0)
    tG, tR, tM = (torch.from_numpy(x).to(dev) for x in (G, R, M))
    from paper_2604_10377_b200 import _lib
    import ctypes as C
    ctx = _lib.context(0)
    out = torch.empty_like(tG)
    rep = _lib.ReportC()
    o = fm.SolverOptions(compute_residual=False).to_c()
    P = lambda x: C.c_void_p(x.data_ptr())  # noqa: E731
    st = ctx._lib.fmap_solve_f32_dev(ctx.handle, 4, 120, P(tG), P(tR), P(tM), 100.0, C.byref(o), P(out), C.byref(rep))
    assert st == 0
    assert 0.0 < rep.factor_seconds < rep.wall_seconds
