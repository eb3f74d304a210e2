"""Back-to-back repetitions of every device entry at BASELINE shapes (hang finder):
    python tools/stress.py [reps]"""
import ctypes as C
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_10377_b200 as fm  # noqa: E402
from paper_2604_10377_b200 import _lib, synth  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 100
cfg = synth.CONFIGS["cfg2"]
data = synth.make_batch(cfg)
t = {k: torch.from_numpy(v).cuda() for k, v in data.items()}
opts = fm.SolverOptions(compute_residual=False)
t0 = time.perf_counter()
for i in range(reps):
    fm.pipeline_device(t["phi1"], t["mass1"], t["F1"], t["ev1"], t["phi2"], t["mass2"], t["F2"], t["ev2"],
                       lam=cfg.lam, sigma=cfg.sigma, opts=opts)
torch.cuda.synchronize()
print(f"pipeline x{reps}: {(time.perf_counter() - t0) / reps * 1e3:.3f} ms", flush=True)
ctx = _lib.context(0)
P = lambda x: C.c_void_p(x.data_ptr())  # noqa: E731
out = torch.empty(cfg.batch, cfg.k, cfg.d, device="cuda")
t0 = time.perf_counter()
for i in range(5 * reps):
    assert ctx._lib.fmap_project_f32_dev(ctx.handle, cfg.batch, cfg.n_src, cfg.k, cfg.d, P(t["phi1"]),
                                         P(t["mass1"]), P(t["F1"]), P(out)) == 0
torch.cuda.synchronize()
print(f"projection x{5 * reps}: {(time.perf_counter() - t0) / (5 * reps) * 1e3:.3f} ms", flush=True)
G, R, e1, e2 = synth.random_normal_equations(64, 200, 256, 7)
M = fm.build_mask(fm.MaskKind.Resolvent, e1, e2, 0.5)
t0 = time.perf_counter()
for i in range(max(1, reps // 10)):
    fm.solve_host(G.astype(np.float64), R.astype(np.float64), M.astype(np.float64), 100.0, opts, precision="f64")
print(f"f64 x{max(1, reps // 10)}: {(time.perf_counter() - t0) / max(1, reps // 10) * 1e3:.3f} ms", flush=True)
cfg4 = synth.CONFIGS["cfg4"]
d4 = synth.make_batch(cfg4, count=32)
t4 = {k: torch.from_numpy(v).cuda() for k, v in d4.items()}
t0 = time.perf_counter()
for i in range(max(1, reps // 10)):
    fm.pipeline_device(t4["phi1"], t4["mass1"], t4["F1"], t4["ev1"], t4["phi2"], t4["mass2"], t4["F2"], t4["ev2"],
                       lam=cfg4.lam, sigma=cfg4.sigma, bidirectional=True, opts=opts)
torch.cuda.synchronize()
print(f"cfg4 (32 pairs, bidirectional) x{max(1, reps // 10)}: {(time.perf_counter() - t0) / max(1, reps // 10) * 1e3:.3f} ms")
print("stress ok")
