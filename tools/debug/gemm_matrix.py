"""Correctness matrix of the DMMA GEMM over sizes (config/smem forced by env in the caller)."""
import os, sys
sys.path.insert(0, ".")
import torch
import paper_2212_02406_b200 as nnb

bad = 0
for n in [int(v) for v in sys.argv[1:]]:
    g = torch.Generator(device="cuda").manual_seed(0)
    a = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    b = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    ref = a @ b
    errs = []
    for _ in range(3):
        c = nnb.matmul(a, b)
        errs.append(((c - ref).norm() / ref.norm()).item())
    print(os.environ.get("NNB_GEMM_CFG", "auto"), os.environ.get("NNB_GEMM_SMEM_PAD", "0"), n, ["%.1e" % e for e in errs])
