"""Kernel timeline of one 4096^2 factorized solve (config 4) from torch.profiler (CUPTI):
each kernel's start offset and duration, so the format pass and host round trips show."""
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
import paper_2212_02406_b200 as nnb  # noqa: E402
from paper_2212_02406_b200 import workloads as W  # noqa: E402

g = 4096
rp, col, val = W.laplacian_5pt(g)
dev = lambda a: torch.from_numpy(a).cuda()
csr = nnb.Csr(dev(rp), dev(col), dev(val), n=g * g, nnz=col.size)
b = dev(W.rhs(g * g, seed=7))
norm = nnb.Normalization(theta=0.2, valid=True)
for _ in range(3):
    nnb.solve_sparse_factorized(csr, b, 63, norm)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    nnb.solve_sparse_factorized(csr, b, 63, norm)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
for e in ev:
    print(f"{(e.time_range.start - t0) / 1e3:8.3f} ms  {e.time_range.elapsed_us():8.1f} us  {e.name[:90]}")
print(f"span {(ev[-1].time_range.end - t0) / 1e3:.3f} ms over {len(ev)} device events")
if "--host" in sys.argv:  # the CUDA runtime calls on the host (same clock)
    hv = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CPU and e.name.startswith("cu")]
    hv.sort(key=lambda e: e.time_range.start)
    for e in hv:
        print(f"host {(e.time_range.start - t0) / 1e3:8.3f} ms  {e.time_range.elapsed_us():8.1f} us  {e.name[:60]}")
