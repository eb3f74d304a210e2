"""e2e (host C ABI, pinned buffers) at cfg2-like shapes (or --b / --k): residual on/off,
copies on/off (FMAP_DEBUG 2 = no H2D, 4 = no D2H).
    python tools/e2e_probe.py [--b 64] [--k 200]"""
import ctypes as C
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2604_10377_b200 as fm  # noqa: E402
from paper_2604_10377_b200 import _lib, synth  # noqa: E402

import argparse  # noqa: E402
ap = argparse.ArgumentParser()
ap.add_argument("--b", type=int, default=64)
ap.add_argument("--k", type=int, default=200)
ap.add_argument("--dbg", default="0,6")
a = ap.parse_args()
B, K = a.b, a.k
G, R, e1, e2 = synth.random_normal_equations(B, K, 256, 7)
M = fm.build_mask(fm.MaskKind.Resolvent, e1, e2, 0.5)
hG, hR, hM = (torch.from_numpy(x).pin_memory() for x in (G, R, M))
hC = torch.empty_like(hG).pin_memory()
ctx = _lib.context(0)
P = lambda x: C.c_void_p(x.data_ptr())  # noqa: E731
for chunks, dbg in (("r2563", d) for d in a.dbg.split(",")):
    os.environ["FMAP_PIPELINE"] = chunks
    if chunks[0] == "r":
        os.environ["FMAP_PIPELINE_W"] = ",".join(chunks[1:])
    os.environ["FMAP_DEBUG"] = dbg
    for res in (False, True):
        o = fm.SolverOptions(compute_residual=res).to_c()
        rep = _lib.ReportC()
        for _ in range(3):
            ctx._lib.fmap_solve_f32(ctx.handle, B, K, P(hG), P(hR), P(hM), 100.0, C.byref(o), P(hC), C.byref(rep))
        t0 = time.perf_counter()
        for _ in range(40):
            st = ctx._lib.fmap_solve_f32(ctx.handle, B, K, P(hG), P(hR), P(hM), 100.0, C.byref(o), P(hC),
                                         C.byref(rep))
        ms = (time.perf_counter() - t0) * 25
        print(f"chunks={chunks} dbg={dbg} residual={res}: {ms:.3f} ms/step (device span {rep.wall_seconds * 1e3:.3f} ms)"
              f"  st={st} launches={len(ctx.last_launches)}")
