"""NNB_ARITH_OZAKI: FP64 products emulated on the int8 tensor cores (tcgen05.mma
kind::i8, Ozaki scheme II, csrc/ozaki.cu), held to the same parity gate as the DMMA
path (north_star: X within 1e-10 relative Frobenius at equal iteration count,
identical nest counts to reach eps, eps within 1e-6 rel + 1e-13)."""
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


def bound(a, b):
    """Per-element bound of the scheme's truncation (53 bits per row of A and column of B):
    |C - C'| <= 2^-53 * (rowmax|A| * sum_k |b_kj| + sum_k |a_ik| * colmax|B|), doubled for slack."""
    ra = np.abs(a).max(axis=1, keepdims=True)
    cb = np.abs(b).max(axis=0, keepdims=True)
    return 2.0 ** -52 * (ra * np.abs(b).sum(axis=0, keepdims=True) + np.abs(a).sum(axis=1, keepdims=True) * cb)


@pytest.mark.parametrize("m,k,n", [(1, 1, 1), (7, 5, 3), (64, 64, 64), (130, 257, 129), (300, 1000, 520),
                                   (1024, 1024, 1024), (129, 4099, 255)])
def test_ozaki_matmul_within_truncation_bound(m, k, n):
    rng = np.random.default_rng(m * 7 + k)
    a = rng.standard_normal((m, k)) * np.exp(rng.uniform(-3, 3, (m, 1)))
    b = rng.standard_normal((k, n)) * np.exp(rng.uniform(-3, 3, (1, n)))
    exact = (a.astype(np.longdouble) @ b.astype(np.longdouble)) if m * k * n <= 2 ** 28 else None
    with nnb.ozaki_arithmetic():
        c = nnb.matmul(a, b)
    ref = nnb.matmul(a, b)  # DMMA
    assert rel_frob(c, ref) < 1e-14, rel_frob(c, ref)
    if exact is not None:
        err = np.abs(c.astype(np.longdouble) - exact).astype(np.float64)
        # + the (compensated) FP64 Horner's final rounding
        lim = bound(a, b) + 2.0 ** -52 * np.abs(exact).astype(np.float64) + 1e-300
        assert np.all(err <= lim), float(np.max(err / lim))


def test_ozaki_matmul_special_values():
    rng = np.random.default_rng(1)
    a, b = rng.standard_normal((200, 300)), rng.standard_normal((300, 150))
    a[5, :] = 0.0  # zero row: exact zeros
    b[:, 7] *= 1e-300  # tiny column (exponent far below 2^-1000)
    a[9, :] *= 1e200
    with nnb.ozaki_arithmetic():
        c = nnb.matmul(a, b)
    ref = a.astype(np.longdouble) @ b.astype(np.longdouble)
    assert np.all(c[5] == 0.0)
    scale = np.abs(a).max(1, keepdims=True) * np.abs(b).sum(0, keepdims=True)
    keep = np.arange(200) != 5
    rel = np.abs(c - ref.astype(np.float64))[keep] / scale[keep]
    assert float(rel.max()) < 1e-15
    a[3, 4] = np.nan  # check_finite (proj/src/kernels.cpp:14-17): DomainError, as on the DMMA path
    with pytest.raises(nnb.DomainError):
        nnb.matmul(a, b)
    with nnb.ozaki_arithmetic(), pytest.raises(nnb.DomainError):
        nnb.matmul(a, b)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_ozaki_chain_matches_reference_nest_counts(port, p):
    """kappa 1e3, N=640 (above the cooperative small-chain size), tolerance stop 1e-12:
    identical nest counts and eps history; X within 1e-10 of the reference."""
    a = W.spd_conditioned(640, 1e3, seed=40 + p)
    x0 = W.x0_transpose_norm(a)
    xr, hr, ir = port.chain(a, x0, p, 80, tol=1e-12)
    with nnb.ozaki_arithmetic():
        x, rep = nnb.nn_chain(a, x0, p=p, max_iters=80, tol=1e-12, order=nnb.ORDER_REFERENCE)
    assert rep.iters == ir and rep.stopped_reason == "tolerance"
    eps_close([e for _, e in rep.history], hr)
    assert rel_frob(x, xr.real) < TOL_X


def test_ozaki_chain_northstar_order_fixed_count(port):
    a = W.gram_shifted(1000, seed=9, shift=1.0)
    x0 = W.x0_transpose_norm(a)
    xr, hr, _ = port.chain(a, x0, 2, 5)
    with nnb.ozaki_arithmetic():
        x, rep = nnb.nn_chain(a, x0, p=2, max_iters=5)
    eps_close([e for _, e in rep.history], hr)
    assert rel_frob(x, xr.real) < TOL_X


def test_ozaki_chain_divergence_index(port):
    from oracle import OracleError

    a = W.gram_shifted(1024, seed=4, shift=1.0)
    x0 = 3.0 * np.eye(1024)
    with pytest.raises(OracleError) as er:
        port.chain(a, x0, 1, 40)
    with nnb.ozaki_arithmetic(), pytest.raises(nnb.DivergenceError) as ed:
        nnb.nn_chain(a, x0, p=1, max_iters=40)
    assert ed.value.nest_index == er.value.index


def test_complex_products_on_the_int8_emulation(port):
    """Complex products under the emulation: 3M over three emulated real products, the
    dual-output DMMA epilogue replaced by elementwise updates (ozaki_arithmetic at small
    sizes; FAST routes complex N >= 3072 products the same way)."""
    rng = np.random.default_rng(12)
    a = rng.standard_normal((300, 260)) + 1j * rng.standard_normal((300, 260))
    b = rng.standard_normal((260, 280)) + 1j * rng.standard_normal((260, 280))
    with nnb.ozaki_arithmetic():
        c = nnb.matmul(a, b)
    assert rel_frob(c, port.matmul(a, b)) < 1e-13
    # a complex Hermitian-positive chain: the emulated chain against the oracle's
    h = rng.standard_normal((400, 200)) + 1j * rng.standard_normal((400, 200))
    az = np.conj(h.T) @ h / 400 + 0.5 * np.eye(200)
    x0 = np.conj(az.T) / (np.abs(az).sum(axis=0).max() * np.abs(az).sum(axis=1).max())
    with nnb.ozaki_arithmetic():
        xz, rz = nnb.nn_chain(az, x0, p=2, max_iters=6)
    xr, hr, _ = port.chain(az, x0, 2, 6)
    assert rel_frob(xz, xr) < 1e-10
    assert np.allclose([e for _, e in rz.history], hr, rtol=1e-6, atol=1e-13)
