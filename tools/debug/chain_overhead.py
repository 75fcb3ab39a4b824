"""Host overhead of nn_chain at config 0 size: wall vs device time for 0/1/30 nests,
X0 built on the device vs given."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2212_02406_b200 as nnb
from paper_2212_02406_b200 import workloads as W

a = torch.from_numpy(W.gram_shifted(256, seed=2212, shift=0.5)).cuda()
x0 = torch.from_numpy(W.x0_transpose_norm(W.gram_shifted(256, seed=2212, shift=0.5))).cuda()
out = torch.empty_like(a)
for label, kw in (("built", {}), ("given", {"x0": x0})):
    for iters in (0, 1, 30):
        args = dict(p=1, max_iters=iters, out=out)
        for _ in range(5):
            nnb.nn_chain(a, kw.get("x0"), **args)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(50):
            x, rep = nnb.nn_chain(a, kw.get("x0"), **args)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / 50 * 1e3
        print("x0=%s iters=%d wall_ms=%.4f device_ms=%.4f" % (label, iters, wall, rep.device_ms))
# python-side overhead: the ctypes call alone vs the wrapper
import cProfile, pstats
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    nnb.nn_chain(a, None, p=1, max_iters=30, out=out)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(12)
