"""Device-entry step time (events around the C-ABI call, as bench.py's `value`) vs the
report's own device span: the per-call host/launch overhead."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2604_10377_b200 as fm  # noqa: E402
from paper_2604_10377_b200 import _lib, synth  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
G, R, e1, e2 = synth.random_normal_equations(B, 200, 256, 7)
M = fm.build_mask(fm.MaskKind.Resolvent, e1, e2, 0.5)
dev = torch.device("cuda", 0)
tG, tR, tM = (torch.from_numpy(x).to(dev) for x in (G, R, M))
C_out = torch.empty_like(tG)
ctx = _lib.context(0)
stream = torch.cuda.Stream(dev)
ctx.set_stream(stream.cuda_stream)
opts = fm.SolverOptions(compute_residual=False).to_c()
P = lambda x: C.c_void_p(x.data_ptr())  # noqa: E731
L, h = ctx._lib, ctx.handle
tot, ker = 0.0, 0.0
n = 40
for it in range(n + 5):
    e0 = torch.cuda.Event(enable_timing=True)
    e1_ = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
    rep = _lib.ReportC()
    st = L.fmap_solve_f32_dev(h, B, 200, P(tG), P(tR), P(tM), 100.0, C.byref(opts), P(C_out), C.byref(rep))
    with torch.cuda.stream(stream):
        e1_.record(stream)
    e1_.synchronize()
    if it >= 5:
        tot += e0.elapsed_time(e1_)
        ker += rep.wall_seconds * 1e3
print(f"b={B}: step {tot / n:.4f} ms, report span {ker / n:.4f} ms, overhead {(tot - ker) / n * 1e3:.1f} us")
