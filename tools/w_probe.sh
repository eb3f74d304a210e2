for w in ${WS:-2,5,6,3 1,5,6,4}; do
  FMAP_PIPELINE=r FMAP_PIPELINE_W=$w python - <<'PY'
import ctypes as C, os, sys, time
sys.path.insert(0, "/root/repo")
import torch
import paper_2604_10377_b200 as fm
from paper_2604_10377_b200 import _lib, synth
G, R, e1, e2 = synth.random_normal_equations(64, 200, 256, 7)
M = fm.build_mask(fm.MaskKind.Resolvent, e1, e2, 0.5)
hG, hR, hM = (torch.from_numpy(x).pin_memory() for x in (G, R, M))
hC = torch.empty_like(hG).pin_memory()
ctx = _lib.context(0)
P = lambda x: C.c_void_p(x.data_ptr())
o = fm.SolverOptions().to_c()
rep = _lib.ReportC()
for _ in range(5):
    ctx._lib.fmap_solve_f32(ctx.handle, 64, 200, P(hG), P(hR), P(hM), 100.0, C.byref(o), P(hC), C.byref(rep))
ts = []
for _ in range(40):
    t0 = time.perf_counter()
    ctx._lib.fmap_solve_f32(ctx.handle, 64, 200, P(hG), P(hR), P(hM), 100.0, C.byref(o), P(hC), C.byref(rep))
    ts.append((time.perf_counter() - t0) * 1e3)
ts.sort()
print(f"W={os.environ['FMAP_PIPELINE_W']}: median {ts[20]:.3f} ms  min {ts[0]:.3f}", flush=True)
PY
done
