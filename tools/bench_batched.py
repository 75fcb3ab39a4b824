"""A/B timing of the batched 16x16 complex kernel variants (NNB_DEBUG=1 NNB_BATCHED_VARIANT=... set by the caller)."""
import os, sys
sys.path.insert(0, ".")
import torch
import paper_2212_02406_b200 as nnb
from paper_2212_02406_b200 import workloads as W

a = W.mimo_gram_device(262144, seed=1)
for _ in range(3):
    x, e = nnb.nn_batched(a, p=2, iters=4)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    x, e = nnb.nn_batched(a, p=2, iters=4)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
idx = torch.arange(0, 262144, 4096, device="cuda")
inv = torch.linalg.inv(a[idx])
rel = (torch.linalg.norm(x[idx] - inv, dim=(1, 2)) / torch.linalg.norm(inv, dim=(1, 2))).max().item()
for _ in range(2):
    xs = nnb.ns_batched(a, 80)
e0.record()
for _ in range(3):
    xs = nnb.ns_batched(a, 80)
e1.record(); torch.cuda.synchronize()
ms_ns = e0.elapsed_time(e1) / 3
print(f"{os.environ.get('NNB_BATCHED_VARIANT','default'):10s} NN {ms:.3f} ms  {262144/ms/1e3:.1f} M inv/s  {262144*11*8*4096/ms/1e9:.2f} TF(4M-equiv, 11 products)  maxrel {rel:.2e}  NS80 {ms_ns:.2f} ms")

# fused detection
h, y, s = W.mimo_uplink_device(262144, seed=2)
for _ in range(3):
    xh, _, _ = nnb.mimo_detect(h, y, 0.1, 2, 4)
e0.record()
for _ in range(10):
    xh, _, _ = nnb.mimo_detect(h, y, 0.1, 2, 4)
e1.record(); torch.cuda.synchronize()
ms_d = e0.elapsed_time(e1) / 10
ser = (torch.sign(xh.real) != torch.sign(s.real)).double().mean().item()
print(f"{'':10s} detect {ms_d:.3f} ms  {262144/ms_d/1e3:.1f} M det/s  sign-err {ser:.2e}")
