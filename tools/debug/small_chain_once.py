"""One config-0 chain (N=256, p=1, 30 nests) for ncu captures of small_chain_kernel."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2212_02406_b200 as nnb
from paper_2212_02406_b200 import workloads as W

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
a = torch.from_numpy(W.gram_shifted(n, seed=2212, shift=0.5)).cuda()
for _ in range(2):
    x, rep = nnb.nn_chain(a, None, p=1, max_iters=30)
torch.cuda.synchronize()
print(rep.device_ms, rep.products)
