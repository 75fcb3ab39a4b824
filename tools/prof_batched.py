"""One C2 batched launch (262144 × 16×16 complex, p=2, 4 nests, Hermitian input) for ncu."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2212_02406_b200 as nnb  # noqa: E402
from paper_2212_02406_b200 import workloads as W  # noqa: E402

a = W.mimo_gram_device(262144, seed=1) if hasattr(W, "mimo_gram_device") else torch.from_numpy(
    W.mimo_gram_host(262144, seed=1)).cuda()
for _ in range(3):
    x, eps = nnb.nn_batched(a, p=2, iters=4)
torch.cuda.synchronize()
print("ok", float(eps.max()))
