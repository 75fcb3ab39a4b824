"""Where a nest's time goes at the C3 size (N=4096, p=2): per-class device time of the
int8 emulation's kernels against the chain's device time (tools/, not part of the bench)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2212_02406_b200 as nnb  # noqa: E402
import bench  # noqa: E402

for n in [int(v) for v in sys.argv[1:]] or [4096]:
    a = bench.dense_inputs(n, seed=1)
    x = nnb.x0(a)
    torch.cuda.synchronize()
    nnb.nn_chain(a, x, p=2, max_iters=10, final_residual=False)
    torch.cuda.synchronize()
    for prof in (False, True):
        nnb.ozaki_profile(prof)
        nnb.ozaki_stats(reset=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _, r = nnb.nn_chain(a, x, p=2, max_iters=10, final_residual=False)
        e1.record()
        torch.cuda.synchronize()
        st = nnb.ozaki_stats(reset=True)
        print(f"n={n} prof={prof}: 10 nests {e0.elapsed_time(e1):.2f} ms (chain device {r.device_ms:.2f} ms)",
              {k: (round(v["ms"], 2), v["launches"]) for k, v in st.items()}, flush=True)
    nnb.ozaki_profile(False)
