"""BASELINE config 4 at its stated size, pinned to the reference offline:
the 4096x4096 Dirichlet 5-point Laplacian + I (N = 16,777,216), b ~ N(0,1) seed 7,
theta = 0.2 (= D^-1), gamma = 63 -- nn::solve_sparse_factorized
(proj/src/factorized.cpp:101-140) run by the reference itself (oracle/_ref, all host threads).
Writes tests/golden/c5_n4096.npz: SHA-256 of x (float64 bytes), 4096 seeded sample entries,
and the spmv count.  Run in the dev container:  python tests/golden/make_golden_c5.py
"""
from __future__ import annotations

import hashlib
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import Reference  # noqa: E402
from paper_2212_02406_b200 import workloads as W  # noqa: E402

OUT = Path(__file__).resolve().parent / "c5_n4096.npz"


def main() -> None:
    os.environ["NN_WORKERS"] = str(os.cpu_count() or 1)
    rp, col, val = W.laplacian_5pt(4096)
    b = W.rhs(4096 * 4096, seed=7)
    t0 = time.perf_counter()
    x, cnt, _ = Reference().sparse_factorized(rp, col, val, b, 63, 0.2)
    print(f"reference solve {time.perf_counter() - t0:.1f} s, spmv {cnt}", flush=True)
    assert not np.any(x.imag)
    xr = np.ascontiguousarray(x.real)
    idx = np.sort(np.random.default_rng(4096).choice(xr.size, 4096, replace=False))
    np.savez_compressed(OUT, x_sha256=hashlib.sha256(xr.tobytes()).hexdigest(), idx=idx, x_sample=xr[idx],
                        spmv=cnt, b_sha256=hashlib.sha256(np.ascontiguousarray(b).tobytes()).hexdigest())
    print("wrote", OUT, hashlib.sha256(xr.tobytes()).hexdigest())


if __name__ == "__main__":
    main()
