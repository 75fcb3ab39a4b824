"""Pinned host<->device copy bandwidth on this box: H2D, D2H, and both at once (two streams)."""
import torch

n = 1 << 27  # 1 GiB of float64
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(2):
    d_a.copy_(h_in, non_blocking=True)
    h_out.copy_(d_b, non_blocking=True)
torch.cuda.synchronize()
gb = n * 8 / 1e9
for name, fn in (("H2D", lambda: d_a.copy_(h_in, non_blocking=True)),
                 ("D2H", lambda: h_out.copy_(d_b, non_blocking=True))):
    e0.record(); fn(); e1.record(); torch.cuda.synchronize()
    print(f"{name}: {gb / (e0.elapsed_time(e1) * 1e-3):.1f} GB/s")
torch.cuda.synchronize()
e0.record()
with torch.cuda.stream(s1):
    d_a.copy_(h_in, non_blocking=True)
with torch.cuda.stream(s2):
    h_out.copy_(d_b, non_blocking=True)
s1.synchronize(); s2.synchronize()
e1.record(); torch.cuda.synchronize()
print(f"H2D+D2H concurrently: {2 * gb / (e0.elapsed_time(e1) * 1e-3):.1f} GB/s total")
