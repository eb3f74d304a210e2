"""BASELINE configurations at their stated batch sizes, end to end through the
C ABI (fmap_project_f32_dev / fmap_pipeline_f32_dev), against float64 truth and
the oracle (restated reference solver, oracle/).

The kernels these shapes select are asserted from fmap_last_launches, so the
default cfg2 projection kernel (proj_pair_kernel: CTA-pair tcgen05 3xTF32, TMA-streamed)
and the k > 256 solver variant are the ones under test.  Bars: projection
max|dA| <= 1e-5 * max|A| (f64 truth); solver max|dC| <= 1e-4 * ||C||_max
(north_star) against the oracle's f64 route on the checked pairs; relative
residual ||C G + lambda M.*C - R||_F / ||R||_F <= 1e-5 on EVERY pair.
Reference sweep these follow: proj/tests/acceptance.cpp:98-162.
"""
import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
TOL_REL = 1e-4
RES_REL = 1e-5
_CACHE = {}


def _batch(name, count=None, **over):
    from paper_2604_10377_b200 import synth
    key = (name, count, tuple(sorted(over.items())))
    if key not in _CACHE:
        cfg = synth.CONFIGS[name]
        if over:
            cfg = synth.PairConfig(**{**cfg.__dict__, **over})
        _CACHE[key] = (cfg, synth.make_batch(cfg, count=count))
    return _CACHE[key]


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _proj64(phi, mass, F):
    phi, mass, F = (x.astype(np.float64) for x in (phi, mass, F))
    return np.matmul(np.swapaxes(phi, 1, 2), mass[..., None] * F)


def _check_direction(oracle, Cgpu, A, B, ev_src, ev_tgt, lam, sigma, check_pairs, what):
    b = Cgpu.shape[0]
    for q in range(b):
        G, R = A[q] @ A[q].T, B[q] @ A[q].T
        M = oracle.mask(1, ev_src[q].astype(np.float64), ev_tgt[q].astype(np.float64), sigma)
        Cq = Cgpu[q].astype(np.float64)
        res = np.linalg.norm(Cq @ G + lam * (M * Cq) - R) / np.linalg.norm(R)
        assert res <= RES_REL, f"{what} pair {q}: relative residual {res:.2e}"
        if q in check_pairs:
            ref = oracle.solve(G, R, M, lam).maps
            err = np.abs(Cq - ref).max()
            assert err <= TOL_REL * np.abs(ref).max(), f"{what} pair {q}: max|dC| {err:.3e}"


def _project(fm, b, n, k, d, phi, mass, F):
    t = [_dev(x) for x in (phi, mass, F)]
    out = torch.empty((b, k, d), device="cuda")
    ctx = fm._lib.context(0)
    st = ctx._lib.fmap_project_f32_dev(ctx.handle, b, n, k, d, *(C.c_void_p(x.data_ptr()) for x in t),
                                       C.c_void_p(out.data_ptr()))
    assert st == 0, ctx.last_error()
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.float64), ctx.last_launches


@pytest.mark.parametrize("pair_env, kernel", [(None, "proj_pair_kernel"), ("0", "proj_tma_kernel")])
def test_projection_default_kernel_at_cfg2_shape(fm, monkeypatch, pair_env, kernel):
    # cfg2: 64 pairs, n = 5000, k = 200, d = 256 -> proj_pair_kernel (CTA pairs,
    # tcgen05.mma.cta_group::2 with M = 256: the kernel the pipeline number is made
    # of) or, with FMAP_PROJ_PAIR=0, the one-CTA proj_tma_kernel; all 64 shapes
    # checked against f64.
    if pair_env is not None:
        monkeypatch.setenv("FMAP_PROJ_PAIR", pair_env)
    cfg, data = _batch("cfg2")
    b, n, k, d = cfg.batch, cfg.n_src, cfg.k, cfg.d
    out, launches = _project(fm, b, n, k, d, data["phi1"], data["mass1"], data["F1"])
    assert launches == [kernel], launches
    ref = _proj64(data["phi1"], data["mass1"], data["F1"])
    err = np.abs(out - ref).max(axis=(1, 2))
    scale = np.abs(ref).max(axis=(1, 2))
    assert np.all(err <= 1e-5 * scale), float((err / scale).max())


@pytest.mark.parametrize("b, n, k, d", [(3, 1000, 132, 200), (2, 2048, 256, 256), (5, 700, 200, 36),
                                        (148, 320, 140, 64)])
def test_projection_pair_kernel_shapes(fm, monkeypatch, b, n, k, d):
    # the CTA-pair kernel at the edges of its range (k just above 128, k = 256, d not
    # a multiple of 32 so the channel halves are padded, n not a multiple of the
    # 16-vertex stage, more clusters than fit the GPU at once)
    monkeypatch.setenv("FMAP_PROJ", "tc")
    rng = np.random.default_rng(b * 1000 + k)
    phi = (rng.standard_normal((b, n, k)) / np.sqrt(n)).astype(np.float32)
    mass = (rng.uniform(0.5, 1.5, (b, n)) / n).astype(np.float32)
    F = rng.standard_normal((b, n, d)).astype(np.float32)
    out, launches = _project(fm, b, n, k, d, phi, mass, F)
    assert launches == ["proj_pair_kernel"], launches
    ref = _proj64(phi, mass, F)
    err = np.abs(out - ref).max(axis=(1, 2))
    scale = np.abs(ref).max(axis=(1, 2))
    assert np.all(err <= 1e-5 * scale), float((err / scale).max())


def _pipeline(fm, name, count=None, bidirectional=False, **over):
    cfg, data = _batch(name, count, **over)
    t = {key: _dev(v) for key, v in data.items()}
    cxy, cyx, rep = fm.pipeline_device(t["phi1"], t["mass1"], t["F1"], t["ev1"], t["phi2"], t["mass2"], t["F2"],
                                       t["ev2"], lam=cfg.lam, sigma=cfg.sigma, bidirectional=bidirectional)
    launches = fm._lib.context(0).last_launches
    A = _proj64(data["phi1"], data["mass1"], data["F1"])
    B = _proj64(data["phi2"], data["mass2"], data["F2"])
    return cfg, data, cxy.cpu().numpy(), (cyx.cpu().numpy() if cyx is not None else None), rep, launches, A, B


def test_pipeline_cfg2_full_batch(fm, oracle):
    # headline configuration, BASELINE generator: residual on all 64 pairs, 8 pairs
    # against the oracle's f64 route
    cfg, data, cxy, _, rep, launches, A, B = _pipeline(fm, "cfg2")
    assert launches.count("proj_pair_kernel") == 2 and "chol_tc_kernel" in launches, launches
    _check_direction(oracle, cxy, A, B, data["ev1"], data["ev2"], cfg.lam, cfg.sigma, set(range(0, 64, 8)), "cfg2")
    assert rep.min_rcond > 1e-7


def test_pipeline_cfg5_full_batch(fm, oracle):
    # 128 partial-shape pairs (n 3000 / 6000, slow target spectrum, 20% zeroed channels)
    cfg, data, cxy, _, rep, launches, A, B = _pipeline(fm, "cfg5")
    assert "chol_tc_kernel" in launches
    _check_direction(oracle, cxy, A, B, data["ev1"], data["ev2"], cfg.lam, cfg.sigma, set(range(0, 128, 16)),
                     "cfg5")


def test_pipeline_cfg4_bidirectional_16_pairs(fm, oracle):
    # k = 300 (the 384-thread, one-CTA-per-SM solver variant; G = A A^T itself is
    # rank-deficient since d = 256 < k), both directions, mask(ev2, ev1) = M^T
    cfg, data, cxy, cyx, rep, launches, A, B = _pipeline(fm, "cfg4", count=16, bidirectional=True)
    assert launches.count("chol_tc_kernel") == 2, launches
    _check_direction(oracle, cxy, A, B, data["ev1"], data["ev2"], cfg.lam, cfg.sigma, {0, 5, 10, 15}, "cfg4 xy")
    _check_direction(oracle, cyx, B, A, data["ev2"], data["ev1"], cfg.lam, cfg.sigma, {0, 7, 15}, "cfg4 yx")


@pytest.mark.parametrize("k", [100, 300])
def test_pipeline_cfg3_batch16_n10000(fm, oracle, k):
    # cfg3 sweep points at the stated batch (16) and n = 10000, end to end
    cfg, data, cxy, _, rep, launches, A, B = _pipeline(fm, f"cfg3_k{k}")
    _check_direction(oracle, cxy, A, B, data["ev1"], data["ev2"], cfg.lam, cfg.sigma, {0, 15}, f"cfg3 k={k}")
