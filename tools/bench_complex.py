"""Complex dense chain throughput (4M-equivalent TFLOP/s: 8·N³ per complex product) at N given."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2212_02406_b200 as nnb

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
g = torch.Generator(device="cuda").manual_seed(3)
b = torch.complex(torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g),
                  torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g))
a = b @ b.conj().T / n + torch.eye(n, dtype=torch.complex128, device="cuda")
x0 = (a.conj().T / (a.abs().sum(0).max() * a.abs().sum(1).max())).contiguous()
x, rep = nnb.nn_chain(a, x0, p=2, max_iters=2, final_residual=False)
x, rep = nnb.nn_chain(a, x0, p=2, max_iters=2, final_residual=False)
tf = rep.products * 8.0 * n ** 3 / (rep.device_ms * 1e-3) / 1e12
r = torch.eye(n, dtype=torch.complex128, device="cuda") - a @ x
print(f"complex N={n}: {rep.products} products in {rep.device_ms:.1f} ms = {tf:.2f} TFLOP/s (4M-equivalent); "
      f"eps after 2 nests {(torch.linalg.norm(r) / n ** 0.5).item():.3e}")
