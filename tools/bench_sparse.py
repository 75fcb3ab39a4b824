"""A/B timing of the factorized sparse solve (C5, 4096^2 Laplacian, gamma=63) through the one-shot API.
NNB_DEBUG=1 NNB_SPARSE_COL=32 forces int32 columns (A/B against the default int16 deltas)."""
import os, sys, hashlib
sys.path.insert(0, ".")
import torch
import paper_2212_02406_b200 as nnb
from paper_2212_02406_b200 import workloads as W

grid = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
n = grid * grid
rp, col, val = W.laplacian_5pt(grid)
dev = lambda v: torch.from_numpy(v).cuda()
csr = nnb.Csr(dev(rp), dev(col), dev(val), n=n, nnz=col.size)
b = dev(W.rhs(n, seed=7))
norm = nnb.Normalization(theta=0.2, valid=True)
for _ in range(3):
    x, _ = nnb.solve_sparse_factorized(csr, b, 63, norm)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    x, _ = nnb.solve_sparse_factorized(csr, b, 63, norm)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
h = hashlib.sha256(x.cpu().numpy().tobytes()).hexdigest()[:16]
tag = "col" + os.environ.get("NNB_SPARSE_COL", "16")
print(f"{tag:10s} {ms:.3f} ms/solve  {ms / 63 * 1e3:.1f} us/application  x sha {h}")
