"""Per-application and fixed (format pass) time of the C5 solve: gamma = 1 vs 63."""
import os, sys
sys.path.insert(0, ".")
import torch
import paper_2212_02406_b200 as nnb
from paper_2212_02406_b200 import workloads as W

rp, col, val = W.laplacian_5pt(4096)
n = 4096 * 4096
dev = lambda v: torch.from_numpy(v).cuda()
csr = nnb.Csr(dev(rp), dev(col), dev(val), n=n, nnz=col.size)
b = dev(W.rhs(n, seed=7))
norm = nnb.Normalization(theta=0.2, valid=True)
res = {}
for gamma in (1, 63):
    for _ in range(3):
        nnb.solve_sparse_factorized(csr, b, gamma, norm)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        nnb.solve_sparse_factorized(csr, b, gamma, norm)
    e1.record()
    torch.cuda.synchronize()
    res[gamma] = e0.elapsed_time(e1) / 10
per = (res[63] - res[1]) / 62
print("dict=%s win=%s bytes/nnz=%d solve63=%.3f ms  per-application=%.1f us  fixed=%.3f ms" % (
    os.environ.get("NNB_SPARSE_DICT", "1"), os.environ.get("NNB_DICT_WIN", "1"), nnb.sparse_last_bytes_per_nnz(),
    res[63], per * 1e3, res[1] - per))
