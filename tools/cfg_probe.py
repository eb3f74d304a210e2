"""Device solve of a BASELINE configuration's inputs (bench.py's make_inputs): solve,
factorization and back-substitution times and how many systems needed the exact
rcond estimator.
    python tools/cfg_probe.py [cfg4] [--reps 5]"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2604_10377_b200 as fm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload", nargs="?", default="cfg4")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
dev = torch.device("cuda", 0)
cfg, b, t, G, R, M = bench.make_inputs(a.workload, 0, 1, dev)
opts = fm.SolverOptions(compute_residual=False)
ws, fs, ex = [], [], 0
for i in range(a.reps + 1):
    _, rep = fm.solve_device(G, R, M, lam=cfg.lam, opts=opts)
    if i:
        ws.append(rep.wall_time.total_seconds() * 1e3)
        ex = rep.rcond_exact_systems
print(f"{a.workload}: b={b} k={cfg.k}: solve {sorted(ws)[len(ws) // 2]:.3f} ms, exact-rcond systems {ex} of {b * cfg.k}, "
      f"min rcond {rep.min_rcond:.3e}")
