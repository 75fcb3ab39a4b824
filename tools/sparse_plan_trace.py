"""Timeline of the row-slab plan setup at 4096^2 (world 1, NCCL): NNB_DEBUG=1 NNB_TRACE=1."""
import os
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2212_02406_b200 as nnb  # noqa: E402
from paper_2212_02406_b200 import workloads as W  # noqa: E402

g = int(sys.argv[1]) if len(sys.argv) > 1 else 4096  # 1448: a 4096^2 / 8 slab's rows
rp, col, val = W.laplacian_5pt(g)
n = g * g
dev = lambda a: torch.from_numpy(a).cuda()
csr = nnb.Csr(dev(rp), dev(col), dev(val), n=n, nnz=col.size)
b = dev(W.rhs(n, seed=7))
norm = nnb.Normalization(theta=0.2, valid=True)
comm = nnb.Comm(1, 0, nnb.Comm.unique_id())
for i in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, _ = nnb.solve_sparse_factorized_sharded(comm, csr, n, b, 63, norm)
    torch.cuda.synchronize()
    print(f"one-shot sharded solve {1e3 * (time.perf_counter() - t0):.2f} ms", file=sys.stderr, flush=True)
comm.close()
