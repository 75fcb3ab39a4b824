"""Small fixed workload for ncu captures: one dense nest (N=8192, p=2), one config-0
chain (N=256), one C2 batch, one C5 solve.  Run plainly first (must exit 0), then under ncu with the same arguments."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2212_02406_b200 as nnb
from paper_2212_02406_b200 import workloads as W

which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which in ("all", "dense"):
    a = torch.from_numpy(W.gram_shifted(8192, seed=1, shift=1.0)).cuda()
    x = nnb.x0(a)
    for _ in range(2):
        x, rep = nnb.nn_chain(a, x, p=2, max_iters=1, final_residual=False)
if which in ("all", "c1"):
    # config 0: the device-resident small chain (one cooperative kernel per run)
    a1 = torch.from_numpy(W.gram_shifted(256, seed=2212, shift=0.5)).cuda()
    for _ in range(2):
        x1, rep1 = nnb.nn_chain(a1, None, p=1, max_iters=30)
if which in ("all", "mimo"):
    am = W.mimo_gram_device(262144, seed=1)
    for _ in range(2):
        xm, em = nnb.nn_batched(am, p=2, iters=4)
if which in ("all", "sparse"):
    rp, col, val = W.laplacian_5pt(4096)
    dev = lambda v: torch.from_numpy(v).cuda()
    csr = nnb.Csr(dev(rp), dev(col), dev(val), n=4096 * 4096, nnz=col.size)
    b = dev(W.rhs(4096 * 4096, seed=7))
    for _ in range(2):
        xs, _ = nnb.solve_sparse_factorized(csr, b, 63, nnb.Normalization(theta=0.2, valid=True))
torch.cuda.synchronize()
print("prof_drive ok", which)
if which == "detect":
    h, y, s = W.mimo_uplink_device(262144, seed=2)
    for _ in range(2):
        xh, _, _ = nnb.mimo_detect(h, y)
    torch.cuda.synchronize()
    print("prof_drive ok detect")
if which == "dense32k":
    # the headline workload: one nest of BASELINE config 3 (N=32768, p=2)
    g = torch.Generator(device="cuda").manual_seed(2212)
    b = torch.randn((32768, 32768), dtype=torch.float64, device="cuda", generator=g)
    a = nnb.matmul_nt(b, b)
    del b
    a = nnb._axpby(1.0 / 32768, a, 0.0, None, 1.0)
    x = nnb.x0(a)
    x, rep = nnb.nn_chain(a, x, p=2, max_iters=1, final_residual=False)
    torch.cuda.synchronize()
    print("prof_drive ok dense32k", rep.device_ms)
