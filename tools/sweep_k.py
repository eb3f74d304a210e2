"""Solver kernel time across k (BASELINE cfg3 resolutions), b pairs each.
    python tools/sweep_k.py [--b 16] [--d 256]"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2604_10377_b200 as fm  # noqa: E402
from paper_2604_10377_b200 import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--b", type=int, default=16)
    ap.add_argument("--d", type=int, default=256)
    ap.add_argument("--ks", default="20,40,60,80,100,120,140,160,180,200,220,240,260,280,300")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    opts = fm.SolverOptions(compute_residual=False)
    print("k,b,kernel_ms,fmaps_per_s,tflops")
    for k in (int(x) for x in a.ks.split(",")):
        G, R, e1, e2 = synth.random_normal_equations(a.b, k, a.d, 3)
        tG, tR, t1, t2 = (torch.from_numpy(x).to(dev) for x in (G, R, e1, e2))
        M = torch.from_numpy(fm.build_mask(fm.MaskKind.Resolvent, e1, e2, 0.5)).to(dev)
        ts = []
        for _ in range(6):
            _, rep = fm.solve_device(tG, tR, M, lam=100.0, opts=opts)
            ts.append(rep.wall_time.total_seconds() * 1e3)
        ms = sorted(ts[1:])[len(ts[1:]) // 2]
        flops = a.b * (k ** 4 / 3 + k ** 3)
        print(f"{k},{a.b},{ms:.4f},{a.b / (ms * 1e-3):.1f},{flops / (ms * 1e-3) / 1e12:.3f}")


if __name__ == "__main__":
    main()
