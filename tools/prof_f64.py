"""ncu driver for the f64 route: cfg2-shaped f64 solve on device-resident inputs.

    python tools/prof_f64.py [--k 200] [--b 64] [--reps 2]
"""
import argparse
import ctypes as C
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2604_10377_b200 import _lib, fmsolve, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--k", type=int, default=200)
    ap.add_argument("--b", type=int, default=64)
    ap.add_argument("--d", type=int, default=256)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    G, R, e1, e2 = synth.random_normal_equations(a.b, a.k, a.d, 7)
    M = fmsolve.build_mask(fmsolve.MaskKind.Resolvent, e1, e2, 0.5)
    dev = torch.device("cuda", 0)
    tG, tR, tM = (torch.from_numpy(x).to(dev).double().contiguous() for x in (G, R, M))
    out = torch.empty_like(tG)
    ctx = _lib.context(0)
    o = fmsolve.SolverOptions(compute_residual=False, rcond_threshold=-1.0).to_c()
    P = lambda x: C.c_void_p(x.data_ptr())  # noqa: E731
    for _ in range(a.reps):
        t0 = time.perf_counter()
        rep = _lib.ReportC()
        st = ctx._lib.fmap_solve_f64_dev(ctx.handle, a.b, a.k, P(tG), P(tR), P(tM), 100.0, C.byref(o), P(out),
                                         C.byref(rep))
        assert st == 0, ctx.last_error()
        print(f"f64 solve: {(time.perf_counter() - t0) * 1e3:.2f} ms wall, {rep.wall_seconds * 1e3:.2f} ms kernel")


if __name__ == "__main__":
    main()
