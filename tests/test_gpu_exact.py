"""Reference-exact arithmetic mode: the dense path BIT-IDENTICAL to the reference (real data).

nnb.reference_arithmetic() switches products to ascending-k explicitly rounded
CUDA-core loops, the Frobenius sum to a serial row-major sum and the nest to the
reference's own P/S/Horner sequence; every assertion here is exact equality.
(The fast DMMA mode is held to the north_star tolerance in test_gpu_parity.py.)"""
import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu
nnb = pytest.importorskip("paper_2212_02406_b200")
from paper_2212_02406_b200 import workloads as W  # noqa: E402


def test_exact_matmul_and_residual(ref):
    rng = np.random.default_rng(1)
    with nnb.reference_arithmetic():
        for (m, k, n) in [(1, 1, 1), (7, 5, 3), (65, 130, 33), (256, 256, 256)]:
            a, b = rng.standard_normal((m, k)), rng.standard_normal((k, n))
            assert np.array_equal(nnb.matmul(a, b), ref.matmul(a, b)[0].real)
        a = W.gram_shifted(200, 2, 0.5)
        x = W.x0_transpose_norm(a)
        assert nnb.residual_epsilon(x, a) == ref.residual_eps(x, a)
    assert nnb.lib().nnb_get_arithmetic() == 0  # restored


def test_exact_steps_and_ns_sum(ref):
    g = golden("steps_spd8.npz")
    wt, z = g["wt"], g["z"]
    with nnb.reference_arithmetic():
        for L in (1, 2, 3, 5):
            assert np.array_equal(nnb.nn_step(z, wt, L), ref.step("nn", z, wt, L)[0].real)
        for L in (1, 2):
            assert np.array_equal(nnb.nn_step(z, wt, L), g[f"nn{L}"])  # golden fixture, bit for bit
        for phi0 in (np.eye(8), 0.9 * np.eye(8)):
            for order in (1, 2, 7, 26):
                assert np.array_equal(nnb.ns_sum(phi0, wt, order)[0], ref.ns_sum(phi0, wt, order)[0].real)


def test_exact_config0_chain(ref):
    """BASELINE config 0 end to end: N=256, Newton, 30 nests — X and the eps history identical."""
    a = W.gram_shifted(256, seed=2212, shift=0.5)
    x0 = W.x0_transpose_norm(a)
    xr, hr, ir, _ = ref.chain(a, x0, 1, 30)
    with nnb.reference_arithmetic():
        x, rep = nnb.nn_chain(a, x0, p=1, max_iters=30, order=nnb.ORDER_REFERENCE)
    assert rep.iters == ir
    assert np.array_equal(x, xr.real)
    assert np.array_equal(np.array([e for _, e in rep.history]), hr)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_exact_tolerance_stop(ref, p):
    a = W.spd_conditioned(160, 1e3, seed=7)
    x0 = W.x0_transpose_norm(a)
    xr, hr, ir, _ = ref.chain(a, x0, p, 60, tol=1e-12)
    with nnb.reference_arithmetic():
        x, rep = nnb.nn_chain(a, x0, p=p, max_iters=60, tol=1e-12)
    assert rep.iters == ir and np.array_equal(x, xr.real)
    assert np.array_equal(np.array([e for _, e in rep.history]), hr)


def test_exact_nn_invert_golden():
    g = golden("nn_invert_spd24.npz")
    norm = nnb.Normalization(theta=float(g["theta"]), valid=True)
    with nnb.reference_arithmetic():
        x, rep = nnb.nn_invert(g["w"], norm, depth_L=2, max_nests=40, tol=1e-12)
    assert np.array_equal(x, g["x"])
    assert np.array_equal(np.array([e for _, e in rep.history]), g["eps"])
