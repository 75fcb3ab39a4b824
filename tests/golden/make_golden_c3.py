"""BASELINE config 2 at its stated size, pinned offline:
N=4096, A = nn::random_spd(4096, 1e3, 3), X0 = A^T/(|A|_1 |A|_inf), depth p = 1, 2, 3,
iterate until eps < 1e-12 (the loop of proj/src/solver.cpp:138-159 with an explicit X0).

Run in the dev container (minutes on 8 cores):
    make -C oracle && python tests/golden/make_golden_c3.py [--ref-first-nest]
It uses the C restatement (oracle/nn_oracle.c), which test_oracle_pins.py pins bit for bit
to the reference compiled in place (matmul real fast path, random_spd, chain).  With
--ref-first-nest it also runs the reference itself (oracle/_ref) for the first p=1 nest at
N=4096 and records that X1 and both eps values agree bit for bit with the port's.
Writes tests/golden/c3_n4096.npz: A's SHA-256, per p the nest count, the eps history,
64 seeded rows x 64 seeded columns of X and ||X||_F.
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

from oracle import Port  # noqa: E402
from paper_2212_02406_b200 import workloads as W  # noqa: E402

OUT = Path(__file__).resolve().parent / "c3_n4096.npz"


def main() -> None:
    port = Port()
    port.set_threads(os.cpu_count() or 1)
    t0 = time.perf_counter()
    a = port.random_spd(4096, 1e3, 3)
    print(f"random_spd(4096) {time.perf_counter() - t0:.1f} s", flush=True)
    sha = hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
    x0 = W.x0_transpose_norm(a)
    rng = np.random.default_rng(2212)
    rows = np.sort(rng.choice(4096, 64, replace=False))
    cols = np.sort(rng.choice(4096, 64, replace=False))
    out = dict(a_sha256=sha, rows=rows, cols=cols, x0_scale=x0[0, 0] / a[0, 0] if a[0, 0] else 0.0,
               x0_sha256=hashlib.sha256(np.ascontiguousarray(x0).tobytes()).hexdigest())
    for p in (1, 2, 3):
        t0 = time.perf_counter()
        x, hist, iters = port.chain(a, x0, p, 80, tol=1e-12)
        xr = x.real
        print(f"p={p}: {iters} nests, eps_last {hist[-1]:.3e}, {time.perf_counter() - t0:.1f} s", flush=True)
        out[f"iters_p{p}"] = iters
        out[f"eps_p{p}"] = hist
        out[f"xs_p{p}"] = xr[np.ix_(rows, cols)]
        out[f"xfrob_p{p}"] = float(np.linalg.norm(xr))
    if "--ref-first-nest" in sys.argv:
        from oracle import Reference

        os.environ["NN_WORKERS"] = str(os.cpu_count() or 1)
        t0 = time.perf_counter()
        xr1, hr1, ir1, _ = Reference().chain(a, x0, 1, 1)
        xp1, hp1, ip1 = port.chain(a, x0, 1, 1)
        out["ref_first_nest_bitexact"] = bool(np.array_equal(xr1, xp1) and np.array_equal(hr1, hp1))
        out["ref_first_nest_eps"] = hr1
        print(f"reference first nest: {time.perf_counter() - t0:.1f} s, bit-exact {out['ref_first_nest_bitexact']}",
              flush=True)
    np.savez_compressed(OUT, **out)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
