"""A small workload over every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck, one tool per run):

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_subset.py

Covers: the cooperative small chain (hand-rolled grid barrier), the launch-per-product
chain (DMMA GEMM configurations incl. the K-split acc_in path through the host-buffer
stream), the 3M complex product, the batched and detect kernels, the sparse dictionary
builds (pair and row dictionaries, incl. a > 255-pair operator that overflows the pair
dictionary), the emulated sharded chains, the generators and the int8 emulation
(tcgen05, small sizes)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2212_02406_b200 as nnb  # noqa: E402
from paper_2212_02406_b200 import workloads as W  # noqa: E402

rng = np.random.default_rng(0)
# dense chains: cooperative small chain (N <= 384), launch-per-product chain
a = W.gram_shifted(96, seed=1, shift=0.5)
nnb.nn_chain(a, None, p=2, max_iters=4, tol=1e-12)
a = W.gram_shifted(520, seed=2, shift=1.0)
nnb.nn_chain(a, None, p=2, max_iters=2)
nnb.nn_chain(a, None, p=1, max_iters=2, order=nnb.ORDER_REFERENCE)
nnb.nn_chain(a, None, p=2, max_iters=2, order=nnb.ORDER_SYMMETRIC)
# GEMM configurations and the K-major variant
for (m, k, n) in [(7, 5, 3), (130, 257, 129), (700, 300, 650)]:
    nnb.matmul(rng.standard_normal((m, k)), rng.standard_normal((k, n)))
nnb.matmul_nt(rng.standard_normal((300, 200)), rng.standard_normal((260, 200)))
# complex 3M product and a complex chain
za = rng.standard_normal((200, 150)) + 1j * rng.standard_normal((200, 150))
zb = rng.standard_normal((150, 180)) + 1j * rng.standard_normal((150, 180))
nnb.matmul(za, zb)
# batched / NS / detect
am = W.mimo_gram_host(70, seed=3)
nnb.nn_batched(am, p=2, iters=4)
nnb.ns_batched(am, 8)
h, y, _ = W.mimo_uplink_host(40, seed=4) if hasattr(W, "mimo_uplink_host") else (None, None, None)
if h is not None:
    nnb.mimo_detect(h, y)
# sparse: Laplacian (row dictionary), wide random operator (> 255 pairs: overflow path)
rp, col, val = W.laplacian_5pt(40)
b = W.rhs(1600, seed=5)
nnb.solve_sparse_factorized(nnb.Csr(rp, col, val, n=1600), b, 15, nnb.Normalization(theta=0.2, valid=True))
n = 600
rows = [np.sort(rng.choice(n, 5, replace=False)) for _ in range(n)]
rp = np.zeros(n + 1, np.int64)
rp[1:] = np.cumsum([len(r) for r in rows])
col = np.concatenate(rows).astype(np.int32)
val = rng.uniform(0.01, 0.1, col.size)
nnb.solve_sparse_factorized(nnb.Csr(rp, col, val, n=n), rng.standard_normal(n), 7,
                            nnb.Normalization(theta=0.2, valid=True))
# emulated sharded chains / sparse slabs
a = W.gram_shifted(300, seed=6, shift=1.0)
nnb.nn_chain_sharded_emulated(a, 3, p=2, max_iters=2)
rp, col, val = W.laplacian_5pt(24)
nnb.solve_sparse_factorized_sharded_emulated(nnb.Csr(rp, col, val, n=576), W.rhs(576, seed=7), 7,
                                             nnb.Normalization(theta=0.2, valid=True), 3)
# generators
nnb.random_spd(40, 1e3, 3)
# int8 emulation (tcgen05 + TMA), small: a product, a chain in symmetric order (upper-tile
# GEMM + mirrored reconstruction) and the sharded schedule (residue blocks, K-block GEMMs
# accumulated mod m, ragged 16-row blocks)
with nnb.ozaki_arithmetic():
    nnb.matmul(rng.standard_normal((200, 300)), rng.standard_normal((300, 260)))
    a = W.gram_shifted(400, seed=8, shift=1.0)
    nnb.nn_chain(a, None, p=2, max_iters=2, order=nnb.ORDER_SYMMETRIC)
    nnb.nn_chain_sharded_emulated(a, 3, p=2, max_iters=2)
torch.cuda.synchronize()
print("sanitize subset ok", nnb.kernel_launches(), "launches")
