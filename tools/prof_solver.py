"""Small driver for ncu: cfg2-shaped solver launches on device-resident inputs.

    python tools/prof_solver.py [--k 200] [--b 64] [--reps 3] [--mode mask|ev]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2604_10377_b200 as fm  # noqa: E402
from paper_2604_10377_b200 import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--k", type=int, default=200)
    ap.add_argument("--b", type=int, default=64)
    ap.add_argument("--d", type=int, default=256)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--mode", default="mask")
    a = ap.parse_args()
    G, R, e1, e2 = synth.random_normal_equations(a.b, a.k, a.d, 7)
    dev = torch.device("cuda", 0)
    tG, tR, t1, t2 = (torch.from_numpy(x).to(dev) for x in (G, R, e1, e2))
    M = torch.from_numpy(fm.build_mask(fm.MaskKind.Resolvent, e1, e2, 0.5)).to(dev)
    opts = fm.SolverOptions(compute_residual=False)
    times, exact = [], []
    for _ in range(a.reps):
        if a.mode == "ev":
            _, rep = fm.solve_device(tG, tR, lam=100.0, ev1=t1, ev2=t2, opts=opts)
        else:
            _, rep = fm.solve_device(tG, tR, M, lam=100.0, opts=opts)
        times.append(rep.wall_time.total_seconds() * 1e3)
        exact.append(getattr(rep, "rcond_exact_systems", -1))
    torch.cuda.synchronize()
    print("solver kernel ms:", " ".join(f"{t:.3f}" for t in times), "| exact-rcond systems:", exact)


if __name__ == "__main__":
    main()
