"""The alternate kernels behind the runtime switches give the
same answers as the default ones: the FP32 SIMT Gram/RHS GEMM and residual kernel
(the fallbacks for shapes the tcgen05 kernels do not serve), the N-split and
one-CTA projection kernels, and the copy-pipelined host entry with equal chunks.
Bars: products and projections against float64 numpy at 1e-5 of their scale;
residuals against the tcgen05 path at 1e-6 relative; maps bitwise.
"""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _normal(fm, A, B):
    import torch
    b, k, d = A.shape
    tA, tB = _dev(A), _dev(B)
    G = torch.empty(b, k, k, device="cuda")
    R = torch.empty(b, k, k, device="cuda")
    ctx = fm._lib.context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    st = ctx._lib.fmap_normal_equations_f32_dev(ctx.handle, b, k, d, C.c_void_p(tA.data_ptr()),
                                                C.c_void_p(tB.data_ptr()), C.c_void_p(G.data_ptr()),
                                                C.c_void_p(R.data_ptr()))
    assert st == 0, ctx.last_error()
    torch.cuda.synchronize()
    launches = ctx.last_launches
    ctx.set_stream(None)
    return G.cpu().numpy().astype(np.float64), R.cpu().numpy().astype(np.float64), launches


@pytest.mark.parametrize("gram", [None, "simt"])
def test_normal_equations_kernels(fm, monkeypatch, gram):
    if gram:
        monkeypatch.setenv("FMAP_GRAM", gram)
    rng = np.random.default_rng(5)
    A = rng.standard_normal((6, 120, 96)).astype(np.float32)
    B = rng.standard_normal((6, 120, 96)).astype(np.float32)
    G, R, launches = _normal(fm, A, B)
    want = "gemm_nt_kernel" if gram else "gram_tc_kernel"
    assert launches and all(x == want for x in launches), launches
    A64, B64 = A.astype(np.float64), B.astype(np.float64)
    Gr = A64 @ np.swapaxes(A64, 1, 2)
    Rr = B64 @ np.swapaxes(A64, 1, 2)
    assert np.abs(G - Gr).max() <= 1e-5 * np.abs(Gr).max()
    assert np.abs(R - Rr).max() <= 1e-5 * np.abs(Rr).max()
    if not gram:
        assert np.array_equal(G, np.swapaxes(G, 1, 2))  # mirrored: exactly symmetric


def _residual(fm, Cm, G, R, M, lam):
    import torch
    b, k, _ = Cm.shape
    t = [_dev(x) for x in (Cm, G, R, M)]
    out = torch.empty(b, dtype=torch.float64, device="cuda")
    ctx = fm._lib.context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    st = ctx._lib.fmap_residual_f32_dev(ctx.handle, b, k, *(C.c_void_p(x.data_ptr()) for x in t),
                                        C.c_float(lam), C.c_void_p(out.data_ptr()))
    assert st == 0, ctx.last_error()
    torch.cuda.synchronize()
    launches = ctx.last_launches
    ctx.set_stream(None)
    return out.cpu().numpy(), launches


def test_residual_simt_matches_tensor_core(fm, monkeypatch):
    rng = np.random.default_rng(9)
    b, k = 5, 72
    Cm, G, R = (rng.standard_normal((b, k, k)).astype(np.float32) for _ in range(3))
    G = (0.5 * (G + np.swapaxes(G, 1, 2))).astype(np.float32)  # a Gram matrix is symmetric
    M = rng.uniform(0.0, 2.0, (b, k, k)).astype(np.float32)
    tc, l1 = _residual(fm, Cm, G, R, M, 3.0)
    monkeypatch.setenv("FMAP_RESIDUAL_SIMT", "1")
    simt, l2 = _residual(fm, Cm, G, R, M, 3.0)
    assert "gram_tc_kernel(residual)" in l1 and "residual_partial_kernel" in l2, (l1, l2)
    C64, G64, R64, M64 = (x.astype(np.float64) for x in (Cm, G, R, M))
    ref = np.sqrt((((C64 @ G64) + 3.0 * M64 * C64 - R64) ** 2).sum(axis=(1, 2)))
    assert np.allclose(tc, ref, rtol=1e-5) and np.allclose(simt, ref, rtol=1e-5)
    assert np.allclose(tc, simt, rtol=1e-6)


@pytest.mark.parametrize("env", [{"FMAP_PROJ_PAIR": "0"}, {"FMAP_PROJ_PAIR": "0", "FMAP_PROJ_SPLIT": "1"},
                                 {"FMAP_PROJ": "simt"}], ids=["one-cta", "n-split", "simt"])
def test_projection_kernels_at_cfg2_shape(fm, monkeypatch, env):
    import torch
    for key, v in env.items():
        monkeypatch.setenv(key, v)
    rng = np.random.default_rng(13)
    b, n, k, d = 8, 2000, 200, 256
    phi = (rng.standard_normal((b, n, k)) / np.sqrt(n)).astype(np.float32)
    mass = (rng.uniform(0.5, 1.5, (b, n)) / n).astype(np.float32)
    F = rng.standard_normal((b, n, d)).astype(np.float32)
    t = [_dev(x) for x in (phi, mass, F)]
    out = torch.empty(b, k, d, device="cuda")
    ctx = fm._lib.context(0)
    st = ctx._lib.fmap_project_f32_dev(ctx.handle, b, n, k, d, *(C.c_void_p(x.data_ptr()) for x in t),
                                       C.c_void_p(out.data_ptr()))
    assert st == 0, ctx.last_error()
    torch.cuda.synchronize()
    want = {"FMAP_PROJ": "project_kernel"}.get(next(iter(env)), "proj_tma_kernel")
    assert ctx.last_launches == [want], ctx.last_launches
    phi64, F64 = phi.astype(np.float64), F.astype(np.float64)
    ref = np.matmul(np.swapaxes(phi64, 1, 2), mass.astype(np.float64)[..., None] * F64)
    err = np.abs(out.cpu().numpy().astype(np.float64) - ref).max(axis=(1, 2))
    assert np.all(err <= 1e-5 * np.abs(ref).max(axis=(1, 2))), float(err.max())


@pytest.mark.parametrize("chunks", ["2", "5", "8"])
def test_host_pipeline_equal_chunks_bitwise(fm, oracle, monkeypatch, chunks):
    # FMAP_PIPELINE=<n> equal chunks (the default weights 2:5:6:3 are covered in
    # test_gpu_solver.py): maps bitwise the unpipelined ones, residual reported.
    from paper_2604_10377_b200 import synth
    G, R, e1, e2 = synth.random_normal_equations(40, 48, 96, 21)
    M = fm.build_mask(fm.MaskKind.Resolvent, e1, e2, 0.5)
    monkeypatch.setenv("FMAP_PIPELINE", chunks)
    piped = fm.solve_host(G, R, M, 100.0)
    assert fm._lib.context(0).last_launches.count("chol_tc_kernel") == int(chunks)
    monkeypatch.setenv("FMAP_PIPELINE", "1")
    plain = fm.solve_host(G, R, M, 100.0)
    assert np.array_equal(piped.maps, plain.maps)
    assert piped.max_residual_norm > 0 and plain.max_residual_norm > 0
