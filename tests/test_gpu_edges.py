"""Edge cases of the CUDA path (GPU only): empty and degenerate shapes, rows
without entries, non-finite inputs — checked against the compiled reference
(oracle/_ref) wherever it defines the answer."""
import numpy as np
import pytest

from conftest import rel_frob

pytestmark = pytest.mark.gpu

nnb = pytest.importorskip("paper_2212_02406_b200")
from paper_2212_02406_b200 import workloads as W  # noqa: E402


def test_gemm_degenerate_shapes(port):
    rng = np.random.default_rng(0)
    a, b = rng.standard_normal((5, 0)), rng.standard_normal((0, 4))
    assert np.array_equal(nnb.matmul(a, b), np.zeros((5, 4)))  # empty inner dimension
    assert nnb.matmul(np.zeros((0, 3)), rng.standard_normal((3, 2))).shape == (0, 2)
    one = nnb.matmul(np.array([[3.0]]), np.array([[-2.5]]))
    assert one.shape == (1, 1) and one[0, 0] == -7.5
    with pytest.raises(nnb.ShapeError):
        nnb.matmul(np.ones((2, 3)), np.ones((2, 3)))


def test_chain_scalar_system(ref):
    """N = 1: the chain is the scalar recurrence x ← x(1 + r + r²), r = 1 − a·x."""
    a = np.array([[4.0]])
    x0 = np.array([[0.1]])
    x, rep = nnb.nn_chain(a, x0, p=2, max_iters=6, order=nnb.ORDER_REFERENCE)
    xr, hr, _, _ = ref.chain(a, x0, 2, 6)
    assert abs(x[0, 0] - 0.25) < 1e-15 and abs(x[0, 0] - xr.real[0, 0]) < 1e-16
    assert rep.iters == 6 and len(rep.history) == 7


def test_chain_zero_iterations_returns_x0():
    a = W.gram_shifted(16, seed=1, shift=1.0)
    x0 = W.x0_transpose_norm(a)
    x, rep = nnb.nn_chain(a, x0, p=2, max_iters=0)
    assert np.array_equal(x, x0) and rep.iters == 0 and rep.products == 1  # the residual only


def test_chain_nonfinite_input_matches_reference_error(ref):
    """A non-finite A: the reference's first residual matmul raises DomainError
    (check_finite, kernels.cpp:14-17) before any nest runs; so does this build."""
    from oracle import OracleError

    a = W.gram_shifted(32, seed=2, shift=1.0)
    a[3, 5] = np.nan
    x0 = W.x0_transpose_norm(np.nan_to_num(a))
    with pytest.raises(OracleError) as er:
        ref.chain(a, x0, 2, 3)
    assert er.value.status == 2  # DomainError in oracle/ref_capi.cpp's status map
    with pytest.raises(nnb.DomainError):
        nnb.nn_chain(a, x0, p=2, max_iters=3)
    # a finite start that blows up inside a nest is a DivergenceError with its 1-based nest index
    with pytest.raises(nnb.DivergenceError) as ed:
        nnb.nn_chain(W.gram_shifted(32, seed=2, shift=1.0), 1e200 * np.eye(32), p=2, max_iters=5)
    assert ed.value.nest_index >= 1


def test_batched_empty_and_single(ref):
    import torch

    empty = torch.empty((0, 16, 16), dtype=torch.complex128, device="cuda")
    x, e = nnb.nn_batched(empty, p=2, iters=4)
    assert x.shape == (0, 16, 16) and e.shape == (0,)
    a = W.mimo_gram_host(1, seed=3)
    x1, e1 = nnb.nn_batched(a, p=2, iters=4)
    xr, er, _ = ref.batched("nn", a, 2, 4)
    assert rel_frob(x1[0], xr[0]) < 1e-10
    h, y, _ = W.mimo_uplink_device(0, seed=1)
    xh, _, _ = nnb.mimo_detect(h, y)
    assert xh.shape[0] == 0


def test_ns_order_zero_and_one(ref):
    w = W.spd_conditioned(8, 10.0, 1)
    w = w / np.trace(w)
    s0, p0 = nnb.ns_sum(np.eye(8), w, 0)
    assert np.array_equal(s0, np.eye(8)) and p0 == 0
    s1, p1 = nnb.ns_sum(np.eye(8), w, 1)
    r1, rp1 = ref.ns_sum(np.eye(8), w, 1)
    assert p1 == rp1 and rel_frob(s1, r1.real) < 1e-15


def test_sparse_rows_without_entries(ref):
    """Rows with no stored entry (the reference's y = 0 for them) and a 1-row operator."""
    n = 50
    rp = np.zeros(n + 1, np.int64)
    cols, vals = [], []
    for i in range(n):
        if i % 7 != 3:  # every 7th row is empty
            for j in (i - 1, i, i + 1):
                if 0 <= j < n:
                    cols.append(j)
                    vals.append(4.0 if j == i else -1.0)
        rp[i + 1] = len(cols)
    col, val = np.array(cols, np.int32), np.array(vals)
    b = np.random.default_rng(4).standard_normal(n)
    norm = nnb.Normalization(theta=0.2, valid=True)
    x, cnt = nnb.solve_sparse_factorized(nnb.Csr(rp, col, val, n=n), b, 31, norm)
    xr, cr, _ = ref.sparse_factorized(rp, col, val, b, 31, 0.2)
    assert cnt == cr == 31 and np.array_equal(x, xr.real)
    one = nnb.Csr(np.array([0, 1], np.int64), np.array([0], np.int32), np.array([5.0]), n=1)
    x1, _ = nnb.solve_sparse_factorized(one, np.array([1.0]), 7, norm)
    x1r, _, _ = ref.sparse_factorized(np.array([0, 1]), np.array([0], np.int32), np.array([5.0]), np.array([1.0]),
                                      7, 0.2)
    assert np.array_equal(x1, x1r.real)


def test_spectral_and_transpose_degenerate():
    assert nnb.conjugate_transpose(np.zeros((0, 5))).shape == (5, 0)
    assert np.array_equal(nnb.random_spd(1, 10.0, 4), np.array([[1.0]]))


def test_fixed_count_chain_stops_at_the_divergent_nest(port):
    """Fixed-count mode: a chain that blows up at nest f raises DivergenceError(f) -- the
    reference's index (proj/src/solver.cpp:151-157, through the bit-exact port) -- and
    stops enqueueing nests two behind the failure instead of running all 40."""
    from oracle import OracleError

    a = W.gram_shifted(1024, seed=4, shift=1.0)
    x0 = 3.0 * np.eye(1024)  # ||I - A X0|| > 1: eps squares every Newton nest until overflow
    with pytest.raises(OracleError) as er:
        port.chain(a, x0, 1, 40)
    f = er.value.index
    assert f is not None and 1 <= f < 20
    l0 = nnb.kernel_launches()
    with pytest.raises(nnb.DivergenceError) as ed:
        nnb.nn_chain(a, x0, p=1, max_iters=40)
    assert ed.value.nest_index == f
    launched = nnb.kernel_launches() - l0
    # (p+1) product launches per nest (+ the residual's), at most kLag = 2 nests past f
    assert launched <= 4 * (f + 3) + 16, launched


def test_release_cached_memory_and_solve_timer():
    """nnb_release_cached_memory trims the library's pool between calls without
    disturbing later work; nnb_sparse_last_solve_ms reports a slab solve's schedule."""
    import paper_2212_02406_b200 as nnb
    from paper_2212_02406_b200 import workloads as W

    a = W.gram_shifted(300, seed=2, shift=1.0)
    x1, _ = nnb.nn_chain(a, None, p=2, max_iters=3)
    nnb.release_cached_memory()
    x2, _ = nnb.nn_chain(a, None, p=2, max_iters=3)
    assert np.array_equal(x1, x2)
    rp, col, val = W.laplacian_5pt(64)
    nnb.solve_sparse_factorized_sharded_emulated(nnb.Csr(rp, col, val, n=4096), W.rhs(4096, seed=1), 15,
                                                 nnb.Normalization(theta=0.2, valid=True), 2)
    assert nnb.sparse_last_solve_ms() > 0.0
