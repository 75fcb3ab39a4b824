"""Where the e2e nest's time goes beyond the device-resident nest (N=32768, p=2)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2212_02406_b200 as nnb  # noqa: E402
import bench  # noqa: E402

n = 32768
a = bench.dense_inputs(n, seed=2212)
x = nnb.x0(a)
torch.cuda.synchronize()
for _ in range(2):
    nnb.nn_chain(a, x, p=2, max_iters=1, final_residual=False)
torch.cuda.synchronize()
t0 = time.perf_counter()
nnb.nn_chain(a, x, p=2, max_iters=1, final_residual=False)
torch.cuda.synchronize()
t_dev = time.perf_counter() - t0
a_h = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
x_h = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
o_h = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
a_h.copy_(a)
x_h.copy_(x)
del a, x
torch.cuda.empty_cache()
an, xn, on = a_h.numpy(), x_h.numpy(), o_h.numpy()
nnb.nn_chain(an, xn, p=2, max_iters=1, final_residual=False, out=on)
t0 = time.perf_counter()
nnb.nn_chain(an, xn, p=2, max_iters=1, final_residual=False, out=on)
t_host = time.perf_counter() - t0
d = torch.empty((n, n), dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
d.copy_(a_h, non_blocking=True)
torch.cuda.synchronize()
t_h2d_contig = time.perf_counter() - t0
t0 = time.perf_counter()
for q in range(8):
    d[:, q * 4096:(q + 1) * 4096].copy_(x_h[:, q * 4096:(q + 1) * 4096], non_blocking=True)
torch.cuda.synchronize()
t_h2d_cols = time.perf_counter() - t0
t0 = time.perf_counter()
o_h.copy_(d, non_blocking=True)
torch.cuda.synchronize()
t_d2h = time.perf_counter() - t0
print(f"device nest {t_dev:.3f} s, host-buffer nest {t_host:.3f} s (+{t_host - t_dev:.3f}); "
      f"H2D 8.6 GB contiguous {t_h2d_contig:.3f} s ({8.6 / t_h2d_contig:.1f} GB/s), column blocks {t_h2d_cols:.3f} s "
      f"({8.6 / t_h2d_cols:.1f} GB/s); D2H {t_d2h:.3f} s")
