"""Projection kernel check + timing: Phi^T diag(Mass) F, cfg2 shapes (b pairs' source
shapes), device-resident; compares against float64 numpy for the first shapes.
    python tools/proj_bench.py [--b 64] [--n 5000] [--k 200] [--d 256]"""
import argparse
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_10377_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--b", type=int, default=64)
    ap.add_argument("--n", type=int, default=5000)
    ap.add_argument("--k", type=int, default=200)
    ap.add_argument("--d", type=int, default=256)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    phi = torch.randn(a.b, a.n, a.k, device=dev, generator=g) / a.n ** 0.5
    mass = torch.rand(a.b, a.n, device=dev, generator=g) / a.n + 0.5 / a.n
    F = torch.randn(a.b, a.n, a.d, device=dev, generator=g)
    out = torch.empty(a.b, a.k, a.d, device=dev)
    ctx = _lib.context(0)
    P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    call = lambda: ctx._lib.fmap_project_f32_dev(ctx.handle, a.b, a.n, a.k, a.d, P(phi), P(mass), P(F), P(out))  # noqa
    assert call() == 0, ctx.last_error()
    torch.cuda.synchronize()
    worst = 0.0
    for q in sorted({0, 1, a.b // 2, a.b - 1}):
        ref = (phi[q].double().T * mass[q].double()) @ F[q].double()
        err = (out[q].double() - ref).abs().max().item() / ref.abs().max().item()
        worst = max(worst, err)
    import time
    for _ in range(2):
        assert call() == 0, ctx.last_error()
    ctx.synchronize() if hasattr(ctx, "synchronize") else torch.cuda.synchronize()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reps = 20
    for _ in range(reps):
        assert call() == 0, ctx.last_error()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3 / reps
    nbytes = 4 * a.b * (a.n * a.k + a.n + a.n * a.d + a.k * a.d)
    print(f"projection b={a.b} n={a.n} k={a.k} d={a.d}: {ms:.3f} ms, {nbytes / ms / 1e6:.0f} GB/s, "
          f"{2 * a.b * a.n * a.k * a.d / ms / 1e9:.1f} TFLOP/s, max rel err vs f64 {worst:.2e} "
          f"({ctx.last_launches})")


if __name__ == "__main__":
    main()
