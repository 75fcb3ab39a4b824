"""Seeded synthetic inputs for the five BASELINE configurations.

There is no public dataset behind the reference (its paper reports no
measurements): every input is synthetic and generated from a
seed with the shapes and distributions BASELINE.json names.  Host generators
use numpy's PCG64 (fast, platform-independent); the large device-side inputs
(C2's channel matrices, C4's 8.6 GB Gram matrix) are generated on the GPU
with torch's seeded Philox generator — setup work outside any timed region.
"""
from __future__ import annotations

import numpy as np


def log_uniform_spectrum(n: int, cond: float) -> np.ndarray:
    """lambda_j = cond^-(n-1-j)/(n-1): log-spaced in [1/cond, 1]
    (the reference's spectrum, proj/src/kernels.cpp:116-124)."""
    if n == 1:
        return np.ones(1)
    t = (n - 1 - np.arange(n)) / (n - 1)
    return cond ** (-t)


def gram_shifted(n: int, seed: int, shift: float) -> np.ndarray:
    """C1/C4: A = B·B^T/n + shift·I, B_ij ~ N(0,1) from `seed` (float64)."""
    b = np.random.default_rng(seed).standard_normal((n, n))
    a = b @ b.T / n
    a = 0.5 * (a + a.T)  # exact symmetry
    a[np.diag_indices(n)] += shift
    return a


def spd_conditioned(n: int, cond: float, seed: int) -> np.ndarray:
    """C3: A = Q·diag(lambda)·Q^T, Q the QR factor of an N(0,1) matrix,
    lambda log-spaced with condition number `cond`."""
    g = np.random.default_rng(seed).standard_normal((n, n))
    q, r = np.linalg.qr(g)
    q *= np.sign(np.diag(r))  # unique Q
    a = (q * log_uniform_spectrum(n, cond)) @ q.T
    return 0.5 * (a + a.T)


def mimo_gram_host(batch: int, seed: int, antennas: int = 128, users: int = 16,
                   sigma2: float = 0.1) -> np.ndarray:
    """C2 on the host: A = H^H·H + sigma²·I, H antennas×users, H_ij ~ CN(0, 1/antennas).
    The product is symmetrised so A is stored exactly Hermitian (a GEMM rounds (i, j)
    and (j, i) independently); the batched kernel's mirrored Horner products need it."""
    rng = np.random.default_rng(seed)
    s = np.sqrt(0.5 / antennas)
    h = (rng.standard_normal((batch, antennas, users)) + 1j * rng.standard_normal((batch, antennas, users))) * s
    a = np.conj(np.transpose(h, (0, 2, 1))) @ h
    a = 0.5 * (a + np.conj(np.transpose(a, (0, 2, 1))))  # exactly Hermitian, as H^H·H is
    a += sigma2 * np.eye(users)
    return a


def mimo_gram_device(batch: int, seed: int, antennas: int = 128, users: int = 16, sigma2: float = 0.1,
                     device: str = "cuda", chunk: int = 32768):
    """C2 on the GPU (torch Philox), chunked so H never exceeds ~1 GB; exactly Hermitian
    like mimo_gram_host."""
    import torch

    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    out = torch.empty((batch, users, users), dtype=torch.complex128, device=device)
    s = (0.5 / antennas) ** 0.5
    eye = torch.eye(users, dtype=torch.complex128, device=device) * sigma2
    for b0 in range(0, batch, chunk):
        b1 = min(batch, b0 + chunk)
        re = torch.randn((b1 - b0, antennas, users), dtype=torch.float64, device=device, generator=gen)
        im = torch.randn((b1 - b0, antennas, users), dtype=torch.float64, device=device, generator=gen)
        h = torch.complex(re, im) * s
        g = h.conj().transpose(1, 2) @ h
        out[b0:b1] = 0.5 * (g + g.conj().transpose(1, 2)) + eye  # exactly Hermitian, as H^H·H is
    return out


def mimo_uplink_host(batch: int, seed: int, antennas: int = 128, users: int = 16, sigma2: float = 0.1):
    """Uplink y = H·s + n per system: H ~ CN(0, 1/antennas), QPSK symbols s (unit energy),
    noise n ~ CN(0, sigma2/antennas).  Returns (H, y, s)."""
    rng = np.random.default_rng(seed)
    sh = np.sqrt(0.5 / antennas)
    h = (rng.standard_normal((batch, antennas, users)) + 1j * rng.standard_normal((batch, antennas, users))) * sh
    s = (rng.choice([-1.0, 1.0], (batch, users)) + 1j * rng.choice([-1.0, 1.0], (batch, users))) / np.sqrt(2)
    sn = np.sqrt(0.5 * sigma2 / antennas)
    noise = (rng.standard_normal((batch, antennas)) + 1j * rng.standard_normal((batch, antennas))) * sn
    y = np.einsum("bau,bu->ba", h, s) + noise
    return h, y, s


def mimo_uplink_device(batch: int, seed: int, antennas: int = 128, users: int = 16, sigma2: float = 0.1,
                       device: str = "cuda"):
    """The same uplink on the GPU (torch Philox), for full-size runs."""
    import torch

    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    sh = (0.5 / antennas) ** 0.5
    h = torch.complex(torch.randn((batch, antennas, users), dtype=torch.float64, device=device, generator=gen),
                      torch.randn((batch, antennas, users), dtype=torch.float64, device=device, generator=gen)) * sh
    bits = torch.randint(0, 2, (batch, users, 2), device=device, generator=gen).to(torch.float64) * 2 - 1
    s = torch.complex(bits[..., 0], bits[..., 1]) / 2 ** 0.5
    sn = (0.5 * sigma2 / antennas) ** 0.5
    noise = torch.complex(torch.randn((batch, antennas), dtype=torch.float64, device=device, generator=gen),
                          torch.randn((batch, antennas), dtype=torch.float64, device=device, generator=gen)) * sn
    y = torch.einsum("bau,bu->ba", h, s) + noise
    return h, y, s


def laplacian_5pt(grid: int, shift: float = 1.0):
    """C5: Dirichlet 5-point Laplacian on a grid×grid mesh plus shift·I, CSR with
    ascending columns (row_ptr int64, col int32, val float64).  nnz = 5N − 4·grid."""
    n = grid * grid
    r = np.arange(n, dtype=np.int64)
    i, j = r // grid, r % grid
    # candidate neighbours in ascending column order: up, left, centre, right, down
    cols = np.stack([r - grid, r - 1, r, r + 1, r + grid], axis=1)
    valid = np.stack([i > 0, j > 0, np.ones(n, bool), j < grid - 1, i < grid - 1], axis=1)
    vals = np.broadcast_to(np.array([-1.0, -1.0, 4.0 + shift, -1.0, -1.0]), (n, 5))
    counts = valid.sum(axis=1)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    col = cols[valid].astype(np.int32)
    val = np.ascontiguousarray(vals[valid])
    return row_ptr, col, val


def rhs(n: int, seed: int, k: int = 1) -> np.ndarray:
    b = np.random.default_rng(seed).standard_normal((n, k))
    return b[:, 0].copy() if k == 1 else b


def x0_transpose_norm(a: np.ndarray) -> np.ndarray:
    """Host form of X0 = A^T/(||A||_1 ||A||_inf) (oracle side of parity tests)."""
    n1 = np.abs(a).sum(axis=0).max()
    ninf = np.abs(a).sum(axis=1).max()
    return a.T * (1.0 / (n1 * ninf))


def x0_jacobi(a: np.ndarray) -> np.ndarray:
    """Host form of X0 = diag(A)^-1."""
    return np.diag(1.0 / np.diag(a))
