"""Per-run device time of nn_chain (p=1, 30 nests) over small N, and eps-history agreement
between the cooperative small-chain kernel and the launch-per-product path (set by env in
the caller: NNB_SMALL_CHAIN_MAX=0 disables the small kernel)."""
import os, sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2212_02406_b200 as nnb
from paper_2212_02406_b200 import workloads as W

tag = os.environ.get("NNB_SMALL_CHAIN_MAX", "default") + "_tm" + os.environ.get("NNB_SMALL_TM", "auto")
for n in [int(v) for v in sys.argv[1:]]:
    a = torch.from_numpy(W.gram_shifted(n, seed=2212, shift=0.5)).cuda()
    for p in (1, 3):
        for _ in range(3):
            x, rep = nnb.nn_chain(a, None, p=p, max_iters=30)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(10):
            x, rep = nnb.nn_chain(a, None, p=p, max_iters=30)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / 10 * 1e3
        xt, rt = nnb.nn_chain(a, None, p=p, max_iters=80, tol=1e-12)
        eps = np.array([e for _, e in rep.history])
        np.save("gpurun_out/small_%s_n%d_p%d.npy" % (tag, n, p), np.concatenate([eps, x.cpu().numpy().ravel()]))
        print("max=%s n=%d p=%d wall_ms=%.3f device_ms=%.3f products=%d us/product=%.2f tol_nests=%d tol_products=%d eps_last=%.3e"
              % (tag, n, p, wall, rep.device_ms, rep.products, rep.device_ms * 1e3 / rep.products, rt.iters, rt.products,
                 eps[-1]))
