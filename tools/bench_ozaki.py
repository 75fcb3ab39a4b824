"""Time one real N^3 product through nnb.matmul on the DMMA path and on the int8
emulation (NNB_ARITH_OZAKI), device-resident operands, CUDA events; and the chain nest.

    python tools/bench_ozaki.py [N ...]
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2212_02406_b200 as nnb  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for n in [int(v) for v in sys.argv[1:]] or [4096, 8192, 16384]:
    g = torch.Generator(device="cuda").manual_seed(n)
    a = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
    b = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
    reps = max(1, int(2e12 / n ** 3))
    with nnb.dmma_arithmetic():
        t_d = timed(lambda: nnb.matmul(a, b), reps)
        c_d = nnb.matmul(a, b)
    with nnb.ozaki_arithmetic():
        t_o = timed(lambda: nnb.matmul(a, b), reps)
        c_o = nnb.matmul(a, b)

    rel = (torch.linalg.norm(c_o - c_d) / torch.linalg.norm(c_d)).item()
    f = 2.0 * n ** 3
    print(f"N={n}: DMMA {t_d:.3f} ms ({f / t_d / 1e9:.1f} TF/s)  OZAKI {t_o:.3f} ms ({f / t_o / 1e9:.1f} TF/s, "
          f"{nnb.ozaki_moduli(n)} moduli)  rel diff {rel:.2e}", flush=True)
    del a, b, c_o, c_d
    torch.cuda.empty_cache()
