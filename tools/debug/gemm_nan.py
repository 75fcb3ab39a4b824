import sys
sys.path.insert(0, ".")
import torch
import paper_2212_02406_b200 as nnb
L = nnb.lib()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
g = torch.Generator(device="cuda").manual_seed(0)
a = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
b = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
ref = a @ b
for trial in range(3):
    c = torch.full((n, n), float("nan"), dtype=torch.float64, device="cuda")
    st = L.nnb_gemm_d(a.data_ptr(), n, b.data_ptr(), n, c.data_ptr(), n, n, n, n, None)
    torch.cuda.synchronize()
    nan = torch.isnan(c)
    wrong = (~nan) & ((c - ref).abs() > 1e-9 * ref.abs().max())
    print("status", st, "nan", int(nan.sum()), "wrong", int(wrong.sum()))
    for name, m in (("nan", nan), ("wrong", wrong)):
        if m.any():
            idx = m.nonzero()
            tiles = torch.unique((idx[:, 0] // 64) * 1000 + idx[:, 1] // 64)
            print(" ", name, "tiles", len(tiles), [(int(t) // 1000, int(t) % 1000) for t in tiles[:6]],
                  "rows%64", torch.unique(idx[:, 0] % 64)[:12].tolist(), "cols%64", torch.unique(idx[:, 1] % 64)[:12].tolist())
            # per-tile count of bad elements
            t0 = idx[0]
            tm, tn = int(t0[0]) // 64, int(t0[1]) // 64
            blk = m[tm*64:(tm+1)*64, tn*64:(tn+1)*64]
            print("   first tile", (tm, tn), "bad in tile", int(blk.sum()), "rows", blk.any(1).nonzero().flatten()[:16].tolist())
