import sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2604_10377_b200 as fm
from paper_2604_10377_b200 import synth
dev = torch.device("cuda", 0)
opts = fm.SolverOptions(compute_residual=False)
for (b, k, d) in [(16, 200, 256), (16, 240, 256), (16, 260, 256), (16, 300, 256), (16, 260, 512)]:
    G, R, e1, e2 = synth.random_normal_equations(b, k, d, 3)
    tG, tR = (torch.from_numpy(x).to(dev) for x in (G, R))
    M = torch.from_numpy(fm.build_mask(fm.MaskKind.Resolvent, e1, e2, 0.5)).to(dev)
    for _ in range(2):
        _, rep = fm.solve_device(tG, tR, M, lam=100.0, opts=opts)
    print(f"b={b} k={k} d={d}: {rep.wall_time.total_seconds()*1e3:.3f} ms, exact-rcond systems {rep.rcond_exact_systems} of {b*k}, min rcond {rep.min_rcond:.3e}", flush=True)
# BASELINE cfg4 inputs
cfg = synth.CONFIGS["cfg4"]
print(cfg)
