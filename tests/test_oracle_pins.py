"""Pin the oracle before trusting it (CPU only).

* the plain-C port reproduces the reference (oracle/_ref) BIT-FOR-BIT;
* both reproduce the committed golden fixtures (made by the reference);
* both satisfy the reference's own known-answer tests for the hot path
  (proj/tests/test_solver.cpp, test_factorized.cpp, test_matrix_core.cpp).
"""
import numpy as np
import pytest

from conftest import golden, rel_frob
from paper_2212_02406_b200 import workloads as W


def crand(rng, *shape, complex_=True):
    x = rng.standard_normal(shape)
    return x + 1j * rng.standard_normal(shape) if complex_ else x + 0j


# ------------------------------------------------------------------ port == reference
def test_port_matmul_bitexact(port, ref):
    rng = np.random.default_rng(0)
    for (m, k, n) in [(5, 7, 3), (64, 64, 64), (70, 33, 65)]:
        a, b = crand(rng, m, k), crand(rng, k, n)
        assert np.array_equal(port.matmul(a, b), ref.matmul(a, b)[0])


def test_port_matmul_real_fast_path_bitexact(port, ref):
    """Real operands take the port's blocked 4x16-register path (ascending k per element,
    mul and add rounded separately); it must equal the reference's complex loop bit for
    bit -- ragged shapes, panel tails, signed zeros and denormal-scale entries included."""
    rng = np.random.default_rng(3)
    for (m, k, n) in [(64, 64, 64), (97, 130, 77), (300, 17, 333), (256, 256, 256), (5, 900, 1000)]:
        a, b = rng.standard_normal((m, k)), rng.standard_normal((k, n))
        a[0, :3] = [-0.0, 1e-310, -1e-300]
        b[:2, 0] = [0.0, -0.0]
        pa, ra = port.matmul(a, b), ref.matmul(a, b)[0]
        assert np.array_equal(pa.view(np.uint64), ra.view(np.uint64)), (m, k, n)


def test_port_residual_and_steps_bitexact(port, ref):
    g = golden("steps_spd8.npz")
    wt, z = g["wt"], g["z"]
    assert port.residual_eps(z, wt) == ref.residual_eps(z, wt)
    for L in (0, 1, 2, 3, 5):
        assert np.array_equal(port.nn_step(z, wt, L), ref.step("nn", z, wt, L)[0])


def test_port_ns_sum_bitexact(port, ref):
    g = golden("steps_spd8.npz")
    wt = g["wt"]
    for phi0 in (np.eye(8), 0.9 * np.eye(8)):
        for order in (0, 1, 2, 7, 26):
            assert np.array_equal(port.ns_sum(phi0, wt, order), ref.ns_sum(phi0, wt, order)[0])


def test_port_chain_bitexact(port, ref):
    a = W.gram_shifted(48, seed=1, shift=0.5)
    x0 = W.x0_transpose_norm(a)
    for p in (1, 2, 3):
        xp, hp, ip = port.chain(a, x0, p, 6)
        xr, hr, ir, _ = ref.chain(a, x0, p, 6)
        assert ip == ir == 6
        assert np.array_equal(xp, xr) and np.array_equal(hp, hr)
    # tolerance mode: identical stopping nest
    xp, hp, ip = port.chain(a, x0, 2, 50, tol=1e-12)
    xr, hr, ir, _ = ref.chain(a, x0, 2, 50, tol=1e-12)
    assert ip == ir and np.array_equal(hp, hr)


def test_port_batched_bitexact(port, ref):
    a = W.mimo_gram_host(24, seed=9)
    xp, ep = port.batched("nn", a, 2, 4, threads=3)
    xr, er, _ = ref.batched("nn", a, 2, 4, threads=2)
    assert np.array_equal(xp, xr) and np.array_equal(ep, er)
    xp, _ = port.batched("ns", a, 2, 80, threads=2)
    xr, _, _ = ref.batched("ns", a, 2, 80, threads=1)
    assert np.array_equal(xp, xr)


def test_port_sparse_bitexact(port, ref):
    rp, col, val = W.laplacian_5pt(12)
    b = W.rhs(144, seed=2)
    assert np.array_equal(port.spmv_block(rp, col, val, b), ref.spmv_block(rp, col, val, b))
    for gamma in (1, 3, 15, 63):
        xp, cp = port.sparse_factorized(rp, col, val, b, gamma, 0.2)
        xr, cr, _ = ref.sparse_factorized(rp, col, val, b, gamma, 0.2)
        assert cp == cr == gamma
        assert np.array_equal(xp, xr)


# ------------------------------------------------------------------ golden fixtures
def test_golden_c1(port):
    g = golden("c1_chain_n32_p1.npz")
    x, hist, iters = port.chain(g["a"], g["x0"], 1, int(g["iters"]))
    assert np.array_equal(x.real, g["x"]) and np.array_equal(hist, g["eps"])


def test_golden_steps(port):
    g = golden("steps_spd8.npz")
    for L in (1, 2, 3):
        assert np.array_equal(port.nn_step(g["z"], g["wt"], L).real, g[f"nn{L}"])
    assert np.array_equal(port.ns_sum(np.eye(8), g["wt"], 26).real, g["ns26"])
    # reference identities: nn_step L=1 == newton, L=2 == chebyshev to 1e-13
    assert rel_frob(g["nn1"], g["newton"]) < 1e-13
    assert rel_frob(g["nn2"], g["chebyshev"]) < 1e-13


def test_golden_mimo(port):
    g = golden("c2_mimo16.npz")
    x, eps = port.batched("nn", g["a"], 2, 4)
    assert np.array_equal(x, g["x_nn"]) and np.array_equal(eps, g["eps_nn"])
    xs, _ = port.batched("ns", g["a"], 2, 80)
    assert np.array_equal(xs, g["x_ns80"])
    # NN(4 nests, p=2) is the Neumann series of order 3^5-1 = 242 > 80: more accurate
    assert np.all(g["eps_nn"] < 1e-10)


def test_golden_sparse(port):
    g = golden("c5_lap16.npz")
    x, cnt = port.sparse_factorized(g["row_ptr"], g["col"], g["val"], g["b"], 63, 0.2)
    assert cnt == int(g["spmv"]) == 63
    assert np.array_equal(x.real, g["x"])


def test_golden_nn_invert(ref):
    g = golden("nn_invert_spd24.npz")
    x, rep = ref.nn_invert(g["w"], float(g["theta"]), True, 2, 40, 1e-12)
    assert np.array_equal(x.real, g["x"]) and np.array_equal(rep["history"], g["eps"])
    nests = len(g["eps"]) - 1
    # report counts are taken before the final scale (proj/src/solver.cpp:161-173)
    assert rep["n3"] == nests * 3 and rep["n2"] == nests * 3


# ------------------------------------------------------------------ known answers
def test_known_scalar_recurrences(port, ref):
    # proj/tests/test_solver.cpp:108-132
    z = np.array([[1.0]])
    w = np.array([[0.5]])
    z1 = ref.step("newton", z, w)[0]
    assert z1[0, 0].real == 1.5
    assert ref.step("newton", z1, w)[0][0, 0].real == 1.875
    assert ref.step("chebyshev", z, w)[0][0, 0].real == 1.75
    assert port.nn_step(z, w, 1)[0, 0].real == 1.5
    assert port.nn_step(z, w, 2)[0, 0].real == 1.75


def test_known_ns_sum_diagonal(port):
    # proj/tests/test_solver.cpp:36-45
    s = port.ns_sum(np.eye(2), np.diag([0.25, 0.75]), 3)
    assert abs(s[0, 0].real - (1 + 0.75 + 0.75 ** 2 + 0.75 ** 3)) < 1e-15
    assert abs(s[1, 1].real - (1 + 0.25 + 0.25 ** 2 + 0.25 ** 3)) < 1e-15


def test_known_equivalent_order(ref):
    # proj/tests/test_solver.cpp:297-308 (minus the test-bug line :303)
    from paper_2212_02406_b200 import equivalent_ns_order

    for (i, L, want) in [(1, 2, 8), (2, 2, 26), (3, 1, 15), (3, 2, 80)]:
        assert ref.equivalent_ns_order(i, L) == want == equivalent_ns_order(i, L)
    assert equivalent_ns_order(50, 2) == 2153693963075557766310746


def test_known_series_equivalence(port):
    # recursive NN == NS of order (L+1)^(i+1)-1 (proj/tests/test_solver.cpp:278-295)
    g = golden("steps_spd8.npz")
    wt = g["wt"]
    for L in (1, 2, 3):
        for i in range(3):
            order = (L + 1) ** (i + 1) - 1
            if order > 80:
                break
            x = np.eye(8) + 0j
            for _ in range(i + 1):
                x = port.nn_step(x, wt, L)
            assert rel_frob(x, port.ns_sum(np.eye(8), wt, order)) < 1e-11


def test_known_sparse_identity(port):
    # proj/tests/test_factorized.cpp:150-163: W = I, theta = 1/8
    n = 8
    rp = np.arange(n + 1, dtype=np.int64)
    col = np.arange(n, dtype=np.int32)
    val = np.ones(n)
    b = np.random.default_rng(1).standard_normal(n)
    x, _ = port.sparse_factorized(rp, col, val, b, 15, 1 / 8)
    assert rel_frob(x.real, b * (1 - (7 / 8) ** 16)) < 1e-12


def test_known_errors(port, ref):
    from oracle import OracleError

    rp, col, val = W.laplacian_5pt(4)
    b = np.ones(16)
    for bad in (0, 6):  # PlanError (proj/src/factorized.cpp:13-19)
        with pytest.raises(OracleError) as e:
            ref.sparse_factorized(rp, col, val, b, bad, 0.2)
        assert e.value.status == 5
    with pytest.raises(OracleError) as e:  # divergence (test_factorized.cpp:199-207)
        ref.sparse_factorized(rp, col, val, b, 32767, 1e150)
    assert e.value.status == 3
    with pytest.raises(OracleError) as e:
        port.sparse_factorized(rp, col, val, b, 32767, 1e150)
    assert e.value.status == 3
    w = ref.random_spd(4, 10, 14).real  # test_solver.cpp:198-213
    with pytest.raises(OracleError) as e:
        ref.nn_invert(w, 1e160, True, 2, 64, 1e-10)
    assert e.value.status == 3 and e.value.index >= 1
    with pytest.raises(OracleError) as e:
        ref.nn_invert(w, 0.1, False, 2, 64, 1e-10)
    assert e.value.status == 4


def test_port_gaussian_stream_and_random_spd_bitexact(port, ref):
    """GaussianStream (proj/include/nn/rng.hpp:15-52) and random_spd (proj/src/kernels.cpp:352-381)
    restated in C with row-wise Householder loops: bit-identical to the reference, so the
    port can generate BASELINE config 2's N=4096 input (the reference's column loops would
    take hours there)."""
    for seed in (0, 3, 2 ** 63 + 11):
        assert np.array_equal(port.gaussian(seed, 1001), ref.gaussian(seed, 1001))
    for n, cond, seed in [(1, 1.0, 1), (2, 10.0, 2), (17, 1e3, 3), (64, 1e3, 3), (130, 1e6, 5), (200, 1e3, 3)]:
        w = port.random_spd(n, cond, seed)
        wr = ref.random_spd(n, cond, seed)
        assert np.array_equal(w, wr.real) and not np.any(wr.imag), (n, cond, seed)
