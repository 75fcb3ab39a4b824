"""Repeatability probe for the DMMA GEMM: where do two identical launches differ?"""
import sys
sys.path.insert(0, ".")
import torch
import paper_2212_02406_b200 as nnb

for n in (256, 1024, 2048, 4096):
    g = torch.Generator(device="cuda").manual_seed(0)
    a = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    b = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    torch.cuda.synchronize()
    cs = [nnb.matmul(a, b) for _ in range(4)]
    torch.cuda.synchronize()
    ref = a @ b
    for i in range(1, 4):
        d = (cs[i] != cs[0])
        nd = int(d.sum().item())
        msg = ""
        if nd:
            idx = d.nonzero()
            rows = torch.unique(idx[:, 0] // 64).tolist()[:8]
            cols = torch.unique(idx[:, 1] // 64).tolist()[:8]
            r_in = torch.unique(idx[:, 0] % 64).tolist()[:16]
            msg = f"tile-rows {rows} tile-cols {cols} rows-in-tile {r_in} maxdiff {(cs[i]-cs[0]).abs().max().item():.3e}"
        print(n, i, "ndiff", nd, "relerr", ((cs[i] - ref).norm() / ref.norm()).item(), msg)
