"""NNB_ORDER_SYMMETRIC: mirrored Horner products (GPU only; run with -m gpu).

For A == Aᵀ and X0 == X0ᵀ every Horner product X·S(R)·R of a nest is
symmetric by push-through ((I − XA)^j X = X (I − AX)^j), so it computes only
its upper tile triangle; R = I − A·X stays a full product.  The bar is the
NORTHSTAR chain's (tests/test_gpu_parity.py): X within 1e-10 relative
Frobenius of the reference oracle at equal nest count, identical nest counts
to reach eps, eps history within 1e-6 relative + 1e-13.
"""
import numpy as np
import pytest

from conftest import rel_frob

pytestmark = pytest.mark.gpu

nnb = pytest.importorskip("paper_2212_02406_b200")
from paper_2212_02406_b200 import workloads as W  # noqa: E402

TOL_X = 1e-10


def eps_close(a, b):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, (a.shape, b.shape)
    floor = (a < 1e-12) & (b < 1e-12)
    ok = floor | (np.abs(a - b) <= 1e-6 * b + 1e-13)
    assert ok.all(), np.c_[a, b][~ok]


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device")
    nnb.lib()


# sizes cover every tile configuration the GEMM picks (16/32/64/128 tiles)
# and ragged edge tiles; N <= 384 runs the one-kernel small chain instead
@pytest.mark.parametrize("n,p,iters", [(400, 1, 12), (777, 2, 6), (1100, 3, 4), (2500, 2, 3)])
def test_symmetric_fixed_nests_vs_reference(ref, n, p, iters):
    a = W.gram_shifted(n, seed=n, shift=0.5)
    x0 = W.x0_transpose_norm(a)
    xr, hr, ir, _ = ref.chain(a, x0, p, iters)
    x, rep = nnb.nn_chain(a, None, p=p, max_iters=iters, order=nnb.ORDER_SYMMETRIC)
    assert rep.iters == ir == iters
    assert rep.products == iters * (p + 1) + 1  # the reference's tally, whatever each product costs
    eps_close([e for _, e in rep.history], hr)
    assert rel_frob(x, xr.real) < TOL_X
    assert np.array_equal(x, x.T)  # mirrored products; at the floor a full nest leaves X unchanged


@pytest.mark.parametrize("p", [1, 2, 3])
def test_symmetric_tolerance_stop_identical_iterations(ref, p):
    a = W.spd_conditioned(520, 1e3, seed=5)
    x0 = W.x0_transpose_norm(a)
    xr, hr, ir, _ = ref.chain(a, x0, p, 60, tol=1e-12)
    x, rep = nnb.nn_chain(a, None, p=p, max_iters=60, tol=1e-12, order=nnb.ORDER_SYMMETRIC)
    assert rep.iters == ir and rep.stopped_reason == "tolerance"
    eps_close([e for _, e in rep.history], hr)
    assert rel_frob(x, xr.real) < TOL_X


def test_symmetric_scaled_identity_start(ref):
    """phi0 = theta·I (nn_invert's start) is a polynomial in A too."""
    a = W.spd_conditioned(640, 50.0, seed=8)
    theta = 1.0 / np.abs(a).sum(1).max()
    x0 = theta * np.eye(640)
    xr, hr, ir, _ = ref.chain(a, x0, 2, 8)
    x, rep = nnb.nn_chain(a, None, p=2, max_iters=8, order=nnb.ORDER_SYMMETRIC,
                          x0_kind=nnb.X0_SCALED_IDENTITY, x0_scale=theta)
    eps_close([e for _, e in rep.history], hr)
    assert rel_frob(x, xr.real) < TOL_X


def test_symmetric_c3_size_matches_northstar():
    """N=4096 (config 2): same nest count to eps < 1e-12 as the full-product
    chain, the same residual floor (the nests below eps 1e-4 run full
    products), X equal to rounding, and X·A ≈ I checked independently."""
    import torch

    a = torch.from_numpy(W.spd_conditioned(4096, 1e3, seed=4)).cuda()
    xs, rs = nnb.nn_chain(a, None, p=2, max_iters=60, tol=1e-12, order=nnb.ORDER_SYMMETRIC)
    xn, rn = nnb.nn_chain(a, None, p=2, max_iters=60, tol=1e-12)
    xs2, rs2 = nnb.nn_chain(a, None, p=2, max_iters=60, tol=1e-12, order=nnb.ORDER_SYMMETRIC)
    torch.cuda.synchronize()
    assert torch.equal(xs, xs2) and rs.history == rs2.history  # run-to-run bit-reproducible
    assert rs.iters == rn.iters and rs.stopped_reason == "tolerance"
    eps_close([e for _, e in rs.history], [e for _, e in rn.history])
    assert (torch.linalg.norm(xs - xn) / torch.linalg.norm(xn)).item() < TOL_X
    r = torch.eye(4096, dtype=torch.float64, device="cuda") - xs @ a
    assert (torch.linalg.norm(r) / 64).item() < 1e-11


def test_symmetric_host_streaming():
    """Host buffers at n >= 8192 take the streamed path; the symmetric order
    runs there too and matches the device-resident NORTHSTAR chain."""
    import torch

    n = 8192
    a = torch.from_numpy(W.gram_shifted(n, seed=9, shift=1.0))
    xs, rs = nnb.nn_chain(a.numpy(), None, p=1, max_iters=3, order=nnb.ORDER_SYMMETRIC)
    xn, rn = nnb.nn_chain(a.cuda(), None, p=1, max_iters=3)
    xn = xn.cpu().numpy()
    eps_close([e for _, e in rs.history], [e for _, e in rn.history])
    assert rel_frob(xs, xn) < TOL_X


def test_symmetric_given_and_jacobi_start(ref):
    """Any symmetric X0 qualifies: a caller's, and diag(A)^-1 (config 1's start)."""
    a = W.gram_shifted(600, seed=12, shift=3.0)  # rho(I - D^-1 A) < 1: Jacobi converges
    for x0, kind in ((W.x0_transpose_norm(a) * 0.9, nnb.X0_GIVEN), (np.diag(1.0 / np.diag(a)), nnb.X0_JACOBI)):
        xr, hr, ir, _ = ref.chain(a, x0, 2, 7)
        x, rep = nnb.nn_chain(a, x0 if kind == nnb.X0_GIVEN else None, p=2, max_iters=7,
                              order=nnb.ORDER_SYMMETRIC, x0_kind=kind)
        eps_close([e for _, e in rep.history], hr)
        assert rel_frob(x, xr.real) < TOL_X
        assert hr[-1] < 1e-3 * hr[0]


def test_symmetric_preconditions():
    a = W.spd_conditioned(300, 10.0, seed=1)
    b = a.copy()
    b[3, 7] = np.nextafter(b[3, 7], np.inf)  # one element one ulp off its mirror
    with pytest.raises(nnb.DomainError):
        nnb.nn_chain(b, None, p=1, max_iters=2, order=nnb.ORDER_SYMMETRIC)
    x0 = W.x0_transpose_norm(a)
    x0[0, 1] = np.nextafter(x0[0, 1], np.inf)
    with pytest.raises(nnb.DomainError):
        nnb.nn_chain(a, x0, p=1, max_iters=2, order=nnb.ORDER_SYMMETRIC)
    with pytest.raises(nnb.DomainError):
        nnb.nn_chain(a.astype(np.complex128), None, p=1, max_iters=2, order=nnb.ORDER_SYMMETRIC,
                     x0_kind=nnb.X0_SCALED_IDENTITY, x0_scale=0.01)


def test_symmetric_nonfinite_input_diverges():
    """A NaN mirrored by a NaN is still symmetric; the chain then reports the
    non-finite residual as the reference's error class does."""
    a = W.spd_conditioned(500, 10.0, seed=2)
    a[10, 20] = a[20, 10] = np.nan
    with pytest.raises((nnb.DivergenceError, nnb.DomainError)):
        nnb.nn_chain(a, None, p=1, max_iters=3, order=nnb.ORDER_SYMMETRIC)


def test_symmetric_int8_emulation_runs_upper_tiles():
    """Under the int8 emulation (N >= 3072 in FAST) a symmetric-order Horner product runs
    only the int8 GEMM tiles that meet the upper triangle and the reconstruction mirrors
    them: for nests above the eps switch the int8 work is R (full) + p upper-tile products,
    X stays symmetric bit for bit, and X matches the full-product chain."""
    import torch

    n, p = 4096, 2
    a = torch.from_numpy(W.spd_conditioned(n, 1e3, seed=7)).cuda()
    nnb.ozaki_profile(True)
    try:
        nnb.ozaki_stats(reset=True)
        xs, rs = nnb.nn_chain(a, None, p=p, max_iters=3, order=nnb.ORDER_SYMMETRIC)
        torch.cuda.synchronize()
        ws = nnb.ozaki_stats(reset=True)["gemm"]
        xn, rn = nnb.nn_chain(a, None, p=p, max_iters=3)
        torch.cuda.synchronize()
        wn = nnb.ozaki_stats(reset=True)["gemm"]
    finally:
        nnb.ozaki_profile(False)
    assert ws["launches"] == wn["launches"] > 0
    tm, tn = n // 128, n // 256
    frac = sum(1 for m in range(tm) for c in range(tn) if 128 * m <= 256 * c + 255) / (tm * tn)
    # 3 nests (eps stays far above 1e-4) + the final residual: 3 + 1 full products,
    # 3·p upper-tile ones; equal moduli counts in both chains assumed by the ratio
    expect = (4 + 3 * p * frac) / (4 + 3 * p)
    assert abs(ws["work"] / wn["work"] - expect) < 0.02, (ws["work"] / wn["work"], expect)
    assert torch.equal(xs, xs.T)
    assert (torch.linalg.norm(xs - xn) / torch.linalg.norm(xn)).item() < 1e-12
    assert np.allclose([e for _, e in rs.history], [e for _, e in rn.history], rtol=1e-9, atol=1e-15)
