# cuBLAS DGEMM ceiling (measurement only, not the product path).
import torch, time
torch.backends.cuda.matmul.allow_tf32 = False
for n in (4096, 8192, 16384):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2): c = a @ b
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    reps = 5 if n < 16384 else 2
    e0.record()
    for _ in range(reps): c = a @ b
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"cuBLAS DGEMM n={n}: {2*n**3/ms/1e9:.2f} TFLOP/s ({ms:.2f} ms)")
x = torch.randn(262144, 16, 16, dtype=torch.complex128, device="cuda")
for _ in range(2): y = x @ x
torch.cuda.synchronize(); e0.record()
for _ in range(5): y = x @ x
e1.record(); torch.cuda.synchronize(); ms = e0.elapsed_time(e1)/5
print(f"cuBLAS batched ZGEMM 262144x16^3: {262144*8*16**3/ms/1e9:.2f} TFLOP/s ({ms:.3f} ms)")
