"""Time nnb.matmul (fused-epilogue DMMA GEMM) over square sizes; TF/s per size."""
import os, sys
sys.path.insert(0, ".")
import torch
import paper_2212_02406_b200 as nnb

for n in [int(v) for v in sys.argv[1:]]:
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        nnb.matmul(a, b)
    reps = max(3, int(2e12 / (2 * n ** 3)))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        nnb.matmul(a, b)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print("persist=%s n=%d ms=%.3f TF=%.2f" % (os.environ.get("NNB_GEMM_PERSIST", "1"), n, ms, 2 * n ** 3 / ms / 1e9))
