import torch, time
x = torch.empty(30_720_000 // 4, dtype=torch.float32).pin_memory()
y = torch.empty_like(x, device="cuda")
for _ in range(3): y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): y.copy_(x, non_blocking=True)
e1.record(); e1.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"H2D 30.7 MB: {ms:.3f} ms = {30.72 / ms:.1f} GB/s")
e0.record()
for _ in range(10): x.copy_(y, non_blocking=True)
e1.record(); e1.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"D2H 30.7 MB: {ms:.3f} ms = {30.72 / ms:.1f} GB/s")
