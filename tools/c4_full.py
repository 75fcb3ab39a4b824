"""BASELINE config 3 (C4) as stated: N=32768, A = B·Bᵀ/N + I, X0 = Aᵀ/(‖A‖₁‖A‖∞), NN depth p=2,
12 nests, on one B200 — the int8-emulated chain (NNB_ARITH_FAST) and the DMMA chain side by
side: eps histories, device time, the two X's relative difference and ‖I − A·X‖_F/√N formed
independently by cuBLAS.  Prints one JSON object."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2212_02406_b200 as nnb  # noqa: E402
import bench  # noqa: E402

n, p, nests = 32768, 2, 12
a = bench.dense_inputs(n, seed=2212)
out = {"config": f"C4: N={n}, p={p}, {nests} nests, A = B·B^T/N + I (seed 2212), X0 = A^T/(|A|_1|A|_inf)"}
xs = {}
for name, ctx in (("int8_emulation", nnb.arithmetic(nnb.ARITH_FAST)), ("dmma", nnb.dmma_arithmetic())):
    with ctx:
        x, rep = nnb.nn_chain(a, None, p=p, max_iters=nests)
    torch.cuda.synchronize()
    flops = rep.products * 2.0 * n ** 3
    out[name] = {"device_ms": round(rep.device_ms, 1), "products": rep.products,
                 "tflops": round(flops / (rep.device_ms * 1e-3) / 1e12, 2),
                 "eps_history": [e for _, e in rep.history]}
    xs[name] = x
    print(name, out[name]["device_ms"], out[name]["eps_history"][-3:], file=sys.stderr, flush=True)
d = (torch.linalg.norm(xs["int8_emulation"] - xs["dmma"]) / torch.linalg.norm(xs["dmma"])).item()
out["x_rel_frob_int8_vs_dmma"] = d
del xs["dmma"]
torch.cuda.empty_cache()
nnb.release_cached_memory()
r = torch.eye(n, dtype=torch.float64, device="cuda")
r.addmm_(a, xs["int8_emulation"], alpha=-1.0)
out["eps_cublas_int8_chain"] = (torch.linalg.norm(r) / n ** 0.5).item()
print(json.dumps(out))
