"""Per-class device time of the emulation's kernels in the device-resident nest vs the
host-buffer (e2e) nest at N=32768, p=2: tells whether the e2e overhead is idle time
(waiting on copies), extra work (per-block splits/recon) or slower kernels (clocks)."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2212_02406_b200 as nnb  # noqa: E402
import bench  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
a = bench.dense_inputs(n, seed=2212)
x = nnb.x0(a)
torch.cuda.synchronize()
for _ in range(2):
    nnb.nn_chain(a, x, p=2, max_iters=1, final_residual=False)
torch.cuda.synchronize()
out = {}
nnb.ozaki_profile(True)
nnb.ozaki_stats(reset=True)
t0 = time.perf_counter()
nnb.nn_chain(a, x, p=2, max_iters=1, final_residual=False)
torch.cuda.synchronize()
out["device"] = {"wall_s": time.perf_counter() - t0, **nnb.ozaki_stats(reset=True)}
nnb.ozaki_profile(False)
a_h = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
x_h = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
o_h = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
a_h.copy_(a)
x_h.copy_(x)
del a, x
torch.cuda.empty_cache()
an, xn, on = a_h.numpy(), x_h.numpy(), o_h.numpy()
nnb.nn_chain(an, xn, p=2, max_iters=1, final_residual=False, out=on)
torch.cuda.synchronize()
for prof in (False, True):
    nnb.ozaki_profile(prof)
    nnb.ozaki_stats(reset=True)
    t0 = time.perf_counter()
    nnb.nn_chain(an, xn, p=2, max_iters=1, final_residual=False, out=on)
    torch.cuda.synchronize()
    out["host_prof" if prof else "host"] = {"wall_s": time.perf_counter() - t0, **nnb.ozaki_stats(reset=True)}
nnb.ozaki_profile(False)
print(json.dumps(out, indent=1))
