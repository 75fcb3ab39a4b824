"""Regenerate tests/golden/*.npz from the reference itself (oracle/_ref).

Run in the dev container, where /root/reference exists:
    make -C oracle && python tests/golden/make_golden.py
The fixtures are small (inputs + the reference's outputs) so the parity
suite can pin the oracle port and the GPU path without /root/reference.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import Reference  # noqa: E402
from paper_2212_02406_b200 import workloads as W  # noqa: E402

OUT = Path(__file__).resolve().parent


def main() -> None:
    ref = Reference()
    # 1) C1 in miniature: Gram + 0.5 I, X0 = A^T/(|A|_1 |A|_inf), Newton, 12 nests
    a = W.gram_shifted(32, seed=7, shift=0.5)
    x0 = W.x0_transpose_norm(a)
    x, hist, iters, _ = ref.chain(a, x0, p=1, max_iters=12)
    np.savez_compressed(OUT / "c1_chain_n32_p1.npz", a=a, x0=x0, x=x.real, eps=hist, iters=iters)

    # 2) reference generator + nn_invert (phi0 = I on theta W) at cond 1e4, L=2
    w = ref.random_spd(24, 1e4, 15).real
    theta, contraction, valid = ref.theta_trace(w)
    xi, rep = ref.nn_invert(w, theta, valid, 2, 40, 1e-12)
    np.savez_compressed(OUT / "nn_invert_spd24.npz", w=w, theta=theta, contraction=contraction, x=xi.real,
                        eps=rep["history"], n3=rep["n3"], n2=rep["n2"])

    # 3) nn_step / newton / chebyshev / ns_sum on a normalized SPD matrix
    w8 = ref.random_spd(8, 1e2, 19).real
    th8, _, _ = ref.theta_trace(w8)
    wt = w8 * th8
    z = np.eye(8) * 0.9
    steps = {f"nn{L}": ref.step("nn", z, wt, L)[0].real for L in (1, 2, 3)}
    steps["newton"] = ref.step("newton", z, wt)[0].real
    steps["chebyshev"] = ref.step("chebyshev", z, wt)[0].real
    ns26, n3 = ref.ns_sum(np.eye(8), wt, 26)
    np.savez_compressed(OUT / "steps_spd8.npz", wt=wt, z=z, ns26=ns26.real, ns26_n3=n3, **steps)

    # 4) C2 in miniature: 16 MIMO Gram systems, NN p=2 x4 + NS order 80
    am = W.mimo_gram_host(16, seed=3)
    xm, epsm, _ = ref.batched("nn", am, 2, 4)
    xs, _, _ = ref.batched("ns", am, 2, 80)
    np.savez_compressed(OUT / "c2_mimo16.npz", a=am, x_nn=xm, eps_nn=epsm, x_ns80=xs)

    # 5) C5 in miniature: 16x16 grid Laplacian + I, theta = 0.2, gamma = 63
    rp, col, val = W.laplacian_5pt(16)
    b = W.rhs(256, seed=5)
    xsp, cnt, _ = ref.sparse_factorized(rp, col, val, b, 63, 0.2)
    np.savez_compressed(OUT / "c5_lap16.npz", row_ptr=rp, col=col, val=val, b=b, x=xsp.real, spmv=cnt)
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)


if __name__ == "__main__":
    main()
