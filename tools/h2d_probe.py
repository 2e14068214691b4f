import torch, time
n = 100_000_000
src = torch.empty(n, dtype=torch.int32).pin_memory()
dst = torch.empty(n, dtype=torch.int32, device="cuda")
for _ in range(3):
    dst.copy_(src, non_blocking=True)
torch.cuda.synchronize()
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
a.record(); dst.copy_(src, non_blocking=True); b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b)
print(f"H2D pinned {4*n/1e6:.0f} MB: {ms:.2f} ms = {4*n/ms/1e6:.1f} GB/s")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    a.record(s); dst.copy_(src, non_blocking=True); b.record(s)
torch.cuda.synchronize()
print(f"side stream: {a.elapsed_time(b):.2f} ms")
