"""Seeded synthetic shape pairs with the BASELINE.json configurations' shapes.

SURVEY.md §8(d) recipe (the reference's own generator, bench.hpp:52-93, draws
A and B directly and has no Phi/Mass/F — see SURVEY D4):

* Mass_v ~ U(0.5, 1.5) / n
* X ~ N(0,1) [n x k];  Q R = qr(diag(sqrt(Mass)) X);  Phi = diag(Mass)^(-1/2) Q
  so that Phi^T diag(Mass) Phi = I
* eigenvalues: ev[0] = 0, ev[1:] = sort(U(0,1) * j^2), j = 1..k-1, scaled to max 200
  (cfg5 target side: U(0,1) * j scaled to max 50 — slower growth, partial shapes)
* F ~ N(0,1) [n x d]; cfg5 zeroes the same seeded 20 % of channels on both sides
* pair q uses seed + q (bench.cpp:36 convention); independent streams per array
  via numpy SeedSequence([seed, stream]) so any shard regenerates any pair.

Everything is drawn in float64 and cast to float32.  No public dataset is
used or needed (the paper's datasets are not in the container).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

STREAMS = {"phi1": 0, "F1": 1, "ev1": 2, "mass1": 3, "phi2": 4, "F2": 5, "ev2": 6, "mass2": 7,
           "chan": 8}


@dataclass(frozen=True)
class PairConfig:
    name: str
    batch: int
    k: int
    d: int
    n_src: int
    n_tgt: int
    lam: float = 100.0
    sigma: float = 0.5
    bidirectional: bool = False
    partial: bool = False  # cfg5: slow target spectrum + zeroed channels
    seed: int = 0


# BASELINE.json "configs", in order (1-based names as in SURVEY.md).
CONFIGS = {
    "cfg1": PairConfig("cfg1", 1, 50, 128, 5000, 5000),
    "cfg2": PairConfig("cfg2", 64, 200, 256, 5000, 5000),
    # cfg3 is a k sweep 20..300 step 20 at batch 16, n=10000, d=256
    **{f"cfg3_k{k}": PairConfig(f"cfg3_k{k}", 16, k, 256, 10000, 10000) for k in range(20, 301, 20)},
    "cfg4": PairConfig("cfg4", 256, 300, 256, 8000, 8000, bidirectional=True),
    "cfg5": PairConfig("cfg5", 128, 100, 128, 3000, 6000, partial=True),
}


def _rng(seed: int, stream: str) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(seed), STREAMS[stream]])))


def mass_orthonormal_basis(n: int, k: int, seed: int, side: str):
    """(Phi [n,k], mass [n]) with Phi^T diag(mass) Phi = I."""
    mass = _rng(seed, f"mass{side}").uniform(0.5, 1.5, size=n) / n
    X = _rng(seed, f"phi{side}").standard_normal((n, k))
    sq = np.sqrt(mass)
    Q, _ = np.linalg.qr(sq[:, None] * X)
    phi = Q / sq[:, None]
    return phi, mass


def spectrum(k: int, seed: int, side: str, slow: bool = False) -> np.ndarray:
    j = np.arange(1, k, dtype=np.float64)
    u = _rng(seed, f"ev{side}").uniform(0.0, 1.0, size=k - 1)
    ev = np.concatenate([[0.0], np.sort(u * (j if slow else j * j))])
    top = 50.0 if slow else 200.0
    if ev[-1] > 0:
        ev *= top / ev[-1]
    return ev


def zeroed_channels(d: int, seed: int, frac: float = 0.2) -> np.ndarray:
    n0 = int(np.floor(frac * d + 0.5))
    return np.sort(_rng(seed, "chan").permutation(d)[:n0])


def make_pair(cfg: PairConfig, q: int) -> dict:
    """All float32 arrays of pair q."""
    seed = cfg.seed + q
    phi1, m1 = mass_orthonormal_basis(cfg.n_src, cfg.k, seed, "1")
    phi2, m2 = mass_orthonormal_basis(cfg.n_tgt, cfg.k, seed, "2")
    F1 = _rng(seed, "F1").standard_normal((cfg.n_src, cfg.d))
    F2 = _rng(seed, "F2").standard_normal((cfg.n_tgt, cfg.d))
    if cfg.partial:
        z = zeroed_channels(cfg.d, cfg.seed)
        F1[:, z] = 0.0
        F2[:, z] = 0.0
    ev1 = spectrum(cfg.k, seed, "1")
    ev2 = spectrum(cfg.k, seed, "2", slow=cfg.partial)
    f = np.float32
    return dict(phi1=phi1.astype(f), mass1=m1.astype(f), F1=F1.astype(f), ev1=ev1.astype(f),
                phi2=phi2.astype(f), mass2=m2.astype(f), F2=F2.astype(f), ev2=ev2.astype(f))


def make_batch(cfg: PairConfig, q0: int = 0, count: int | None = None) -> dict:
    """Stacked [b, ...] float32 arrays for pairs q0 .. q0+count-1."""
    count = cfg.batch if count is None else count
    pairs = [make_pair(cfg, q) for q in range(q0, q0 + count)]
    return {key: np.stack([p[key] for p in pairs]) for key in pairs[0]}


def descriptors_f64(pair: dict) -> tuple[np.ndarray, np.ndarray]:
    """A = Phi1^T M1 F1, B = Phi2^T M2 F2 in float64 from the float32 arrays (checker side)."""
    def proj(phi, m, F):
        phi, m, F = (x.astype(np.float64) for x in (phi, m, F))
        return phi.T @ (m[:, None] * F)
    return proj(pair["phi1"], pair["mass1"], pair["F1"]), proj(pair["phi2"], pair["mass2"], pair["F2"])


def random_normal_equations(b: int, k: int, d: int, seed: int, lam_mask: str = "resolvent",
                            sigma: float = 0.5):
    """Cheap solver inputs with the BASELINE statistics but no n-dimension:
    A, B ~ N(0,1)/sqrt(d) (like bench.hpp:78-85), eigenvalues per the recipe.
    Returns float32 (G, R, ev1, ev2) with G = A A^T, R = B A^T computed in
    float64 then rounded."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, 99])))
    A = rng.standard_normal((b, k, d)) / np.sqrt(d)
    B = rng.standard_normal((b, k, d)) / np.sqrt(d)
    G = np.einsum("qkd,qjd->qkj", A, A)
    R = np.einsum("qkd,qjd->qkj", B, A)
    ev1 = np.stack([spectrum(k, seed + q, "1") for q in range(b)])
    ev2 = np.stack([spectrum(k, seed + q, "2") for q in range(b)])
    f = np.float32
    return G.astype(f), R.astype(f), ev1.astype(f), ev2.astype(f)
