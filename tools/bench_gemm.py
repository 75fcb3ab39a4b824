"""GEMM A/B: B row-major [k][n] (linear tile) vs K-major Bᵀ (swizzled tile), CUDA-event timed."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2212_02406_b200 as nnb

for n in [int(v) for v in sys.argv[1:]] or [8192, 16384]:
    g = torch.Generator(device="cuda").manual_seed(0)
    a = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    b = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    bt = b.t().contiguous()
    L = nnb.lib()
    c = torch.empty_like(a)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for name, fn in (("nn", lambda: L.nnb_gemm_d(a.data_ptr(), n, b.data_ptr(), n, c.data_ptr(), n, n, n, n, None)),
                     ("nt", lambda: L.nnb_gemm_nt_d(a.data_ptr(), n, bt.data_ptr(), n, c.data_ptr(), n, n, n, n, None))):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        reps = 5
        e0.record()
        for _ in range(reps):
            fn()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        err = ((c - a @ b).norm() / (a @ b).norm()).item()
        print(f"n={n} {name}: {2*n**3/ms/1e9:.2f} TFLOP/s ({ms:.2f} ms) relerr {err:.1e}")
