"""Timeline of one-nest nn_chain calls on device buffers at N=32768 (NNB_DEBUG=1 NNB_TRACE=1
prints the chain's marks) against a K-nest call: where a one-nest call's extra time goes."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2212_02406_b200 as nnb  # noqa: E402
import bench  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
a = bench.dense_inputs(n, seed=2212)
x = nnb.x0(a)
torch.cuda.synchronize()
for _ in range(2):
    x, _ = nnb.nn_chain(a, x, p=2, max_iters=1, final_residual=False)
torch.cuda.synchronize()
for k in (1, 1, 3):
    t0 = time.perf_counter()
    x, r = nnb.nn_chain(a, x, p=2, max_iters=k, final_residual=False)
    torch.cuda.synchronize()
    print(f"K={k}: wall {1e3 * (time.perf_counter() - t0) / k:.1f} ms per nest, chain device {r.device_ms / k:.1f} ms",
          flush=True)
