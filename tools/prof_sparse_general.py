"""Launch-list driver: the 4096^2 5-point pattern with random off-diagonal values (no
value dictionary applies) through solve_sparse_factorized."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2212_02406_b200 as nnb
from paper_2212_02406_b200 import workloads as W

rp, col, val = W.laplacian_5pt(4096)
rng = np.random.default_rng(11)
off = val != 5.0
val = val.copy()
val[off] = -rng.uniform(0.5, 1.0, int(off.sum()))
b = W.rhs(4096 * 4096, seed=7)
dev = lambda v: torch.from_numpy(v).cuda()
csr = nnb.Csr(dev(rp), dev(col), dev(val), n=4096 * 4096, nnz=col.size)
bb = dev(b)
for _ in range(2):
    x, _ = nnb.solve_sparse_factorized(csr, bb, 63, nnb.Normalization(theta=0.2, valid=True))
torch.cuda.synchronize()
print("ok", nnb.sparse_last_format())
