"""Normal-equations kernel check + timing (cfg2: G = A A^T, R = B A^T, 64 pairs,
k = 200, d = 256), device-resident, CUDA events; max error vs float64.
    python tools/gram_bench.py [--b 64] [--k 200] [--d 256]"""
import argparse
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2604_10377_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--b", type=int, default=64)
    ap.add_argument("--k", type=int, default=200)
    ap.add_argument("--d", type=int, default=256)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    A = torch.randn(a.b, a.k, a.d, device=dev, generator=g)
    B = torch.randn(a.b, a.k, a.d, device=dev, generator=g)
    G = torch.empty(a.b, a.k, a.k, device=dev)
    R = torch.empty_like(G)
    ctx = _lib.context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)  # events below time the library's work
    P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    call = lambda: ctx._lib.fmap_normal_equations_f32_dev(ctx.handle, a.b, a.k, a.d, P(A), P(B), P(G), P(R))  # noqa
    for _ in range(3):
        assert call() == 0, ctx.last_error()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        call()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 20
    Gr = A.double() @ A.double().transpose(1, 2)
    Rr = B.double() @ A.double().transpose(1, 2)
    err = max(((G.double() - Gr).abs().max() / Gr.abs().max()).item(), ((R.double() - Rr).abs().max() / Rr.abs().max()).item())
    print(f"normal equations b={a.b} k={a.k} d={a.d}: {ms * 1e3:.1f} us per call, max rel err {err:.2e} "
          f"({ctx.last_launches})")


if __name__ == "__main__":
    main()
