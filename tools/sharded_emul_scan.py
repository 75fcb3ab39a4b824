"""Device time of one int8-emulated nest run as the G-rank sharded schedule (virtual ranks
one after another on this GPU) against the single-GPU nest: the per-rank compute cost of
the K-block split (tools/, not part of the bench)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2212_02406_b200 as nnb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
worlds = [int(w) for w in sys.argv[2].split(",") if w] if len(sys.argv) > 2 else [1, 2, 4, 8]
g = torch.Generator(device="cuda").manual_seed(1)
b = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
a = nnb.matmul_nt(b, b)
del b
a = nnb._axpby(1.0 / n, a, 0.0, None, 1.0)
x = nnb.x0(a)
torch.cuda.synchronize()
nnb.nn_chain(a, x, p=2, max_iters=1, final_residual=False)
nnb.ozaki_stats(reset=True)
nnb.ozaki_profile(True)
_, r = nnb.nn_chain(a, x, p=2, max_iters=1, final_residual=False)
torch.cuda.synchronize()
st = nnb.ozaki_stats(reset=True)
print(f"single n={n}: {r.device_ms:.1f} ms", {k: (round(v['ms'], 1), v['launches']) for k, v in st.items()}, flush=True)
for w in worlds:
    _, r = nnb.nn_chain_sharded_emulated(a, w, x, p=2, max_iters=1, final_residual=False)
    torch.cuda.synchronize()
    nnb.ozaki_stats(reset=True)
    _, r = nnb.nn_chain_sharded_emulated(a, w, x, p=2, max_iters=1, final_residual=False)
    torch.cuda.synchronize()
    st = nnb.ozaki_stats(reset=True)
    print(f"world {w}: {r.device_ms:.1f} ms", {k: (round(v['ms'], 1), v['launches']) for k, v in st.items()},
          flush=True)
