"""check_stationarity kernel timing at cfg2 (64 pairs, k = 200): fmap_residual_f32_dev,
CUDA events, steady state.     python tools/residual_bench.py"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2604_10377_b200 import _lib  # noqa: E402

b, k = 64, 200
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
Cm, G, R, M = (torch.randn(b, k, k, device=dev, generator=g) for _ in range(4))
out = torch.empty(b, dtype=torch.float64, device=dev)
ctx = _lib.context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)  # events below time the library's work
P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
call = lambda: ctx._lib.fmap_residual_f32_dev(ctx.handle, b, k, P(Cm), P(G), P(R), P(M), C.c_float(100.0), P(out))  # noqa
for _ in range(3):
    assert call() == 0, ctx.last_error()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    call()
e1.record()
e1.synchronize()
print(f"residual b={b} k={k}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us per call ({ctx.last_launches})")
import time  # noqa: E402
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    call()
torch.cuda.synchronize()
print(f"residual (wall, device-synchronized): {(time.perf_counter() - t0) / 20 * 1e6:.1f} us per call")
