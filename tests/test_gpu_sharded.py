"""Row-sharded chain (config 3 path) on the GPU: the emulated multi-rank schedule
(virtual ranks on one device) and the real NCCL path at world size 1."""
import numpy as np
import pytest

from conftest import rel_frob

pytestmark = pytest.mark.gpu
nnb = pytest.importorskip("paper_2212_02406_b200")
from paper_2212_02406_b200 import workloads as W  # noqa: E402


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_emulated_sharded_matches_single_gpu_and_oracle(port, world):
    n = 1000  # ragged: 63 16-row units over 3 or 8 ranks
    a = W.gram_shifted(n, seed=3, shift=1.0)
    x1, r1 = nnb.nn_chain(a, None, p=2, max_iters=8)
    xs, rs = nnb.nn_chain_sharded_emulated(a, world, None, p=2, max_iters=8)
    assert rs.iters == r1.iters == 8 and rs.products == r1.products
    assert rel_frob(xs, x1) < 1e-12
    e1 = np.array([e for _, e in r1.history])
    es = np.array([e for _, e in rs.history])
    assert np.allclose(es, e1, rtol=1e-10, atol=1e-15)
    if world in (1, 3):  # oracle cross-check at a CPU-friendly size
        a2 = W.gram_shifted(264, seed=3, shift=1.0)
        xs2, _ = nnb.nn_chain_sharded_emulated(a2, world, None, p=2, max_iters=8)
        xr, hr, _ = port.chain(a2, W.x0_transpose_norm(a2), 2, 8)
        assert rel_frob(xs2, xr.real) < 1e-10


def test_emulated_sharded_tolerance_stop(ref):
    a = W.spd_conditioned(256, 1e3, seed=5)
    x0 = W.x0_transpose_norm(a)
    xr, hr, ir, _ = ref.chain(a, x0, 2, 60, tol=1e-12)
    xs, rs = nnb.nn_chain_sharded_emulated(a, 4, None, p=2, max_iters=60, tol=1e-12)
    assert rs.iters == ir and rs.stopped_reason == "tolerance"
    assert rel_frob(xs, xr.real) < 1e-10


@pytest.mark.parametrize("kind", [nnb.X0_TRANSPOSE_NORM, nnb.X0_JACOBI, nnb.X0_SCALED_IDENTITY])
def test_nccl_world1_matches_single_gpu(kind):
    import torch

    # strongly diagonally dominant so that the Jacobi start contracts too
    a = W.gram_shifted(512, seed=4, shift=40.0)
    comm = nnb.Comm(1, 0, nnb.Comm.unique_id())
    try:
        scale = 1.0 / np.abs(a).sum(axis=1).max()
        xs, rs = nnb.nn_chain_sharded(comm, a, 512, None, p=2, max_iters=10, x0_kind=kind, x0_scale=scale)
        x1, r1 = nnb.nn_chain(a, None, p=2, max_iters=10, x0_kind=kind, x0_scale=scale)
        assert rel_frob(xs, x1) < 1e-12
        assert np.allclose([e for _, e in rs.history], [e for _, e in r1.history], rtol=1e-10, atol=1e-15)
        # device-resident rows, as bench.py uses them
        ad = torch.from_numpy(a).cuda()
        xd, rd = nnb.nn_chain_sharded(comm, ad, 512, None, p=2, max_iters=10, x0_kind=kind, x0_scale=scale)
        torch.cuda.synchronize()
        assert rel_frob(xd.cpu().numpy(), x1) < 1e-12
    finally:
        comm.close()


def test_sharded_divergence_reported():
    a = W.gram_shifted(64, seed=1, shift=1.0)
    with pytest.raises(nnb.DivergenceError) as e:
        nnb.nn_chain_sharded_emulated(a, 2, None, p=2, max_iters=30, x0_kind=nnb.X0_SCALED_IDENTITY, x0_scale=1e160)
    assert e.value.nest_index >= 1


# ---------------------------------------------------------------- sparse row slabs (config 4 path)
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_sparse_sharded_emulated_bitexact(ref, world):
    """Halo exchange + interior/boundary split: bit-identical to the reference for any world."""
    rp, col, val = W.laplacian_5pt(100)
    b = W.rhs(10000, seed=world)
    csr = nnb.Csr(rp, col, val, n=10000)
    norm = nnb.Normalization(theta=0.2, valid=True)
    xs, cnt = nnb.solve_sparse_factorized_sharded_emulated(csr, b, 63, norm, world)
    # each slab's rows in 1-byte pattern codes; one slab (whole grid rows) runs temporal-blocked
    # passes, the other partitions (16-row units, not whole 100-cell grid rows) one launch per
    # application
    assert nnb.sparse_last_format() == ("row-dictionary-stencil-tb" if world == 1 else "row-dictionary")
    xr, cr, _ = ref.sparse_factorized(rp, col, val, b, 63, 0.2)
    assert cnt == cr == 63 and np.array_equal(xs, xr.real)
    b2 = np.random.default_rng(world).standard_normal((10000, 2))  # two right-hand sides: int16 deltas
    xs2, _ = nnb.solve_sparse_factorized_sharded_emulated(csr, b2, 15, norm, world)
    xr2, _, _ = ref.sparse_factorized(rp, col, val, b2, 15, 0.2)
    assert np.array_equal(xs2, xr2.real)


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_sparse_sharded_temporal_blocking_bitexact(ref, world):
    """Slabs of whole grid rows (64×64 grid: 32, 16 or 8 grid rows per slab) run the
    temporal-blocked passes with a halo of the pass depth exchanged once per pass; x bit-identical to the
    reference.  World 3 (slabs not whole grid rows) keeps one launch per application."""
    rp, col, val = W.laplacian_5pt(64)
    b = W.rhs(4096, seed=20 + world)
    xs, cnt = nnb.solve_sparse_factorized_sharded_emulated(nnb.Csr(rp, col, val, n=4096), b, 63,
                                                           nnb.Normalization(theta=0.2, valid=True), world)
    assert nnb.sparse_last_format() == ("row-dictionary" if world == 3 else "row-dictionary-stencil-tb")
    xr, cr, _ = ref.sparse_factorized(rp, col, val, b, 63, 0.2)
    assert cnt == cr == 63 and np.array_equal(xs, xr.real)


def test_sparse_sharded_emulated_full_size_matches_single():
    import torch

    rp, col, val = W.laplacian_5pt(4096)
    n = 4096 * 4096
    dev = lambda a: torch.from_numpy(a).cuda()
    csr = nnb.Csr(dev(rp), dev(col), dev(val), n=n, nnz=col.size)
    b = dev(W.rhs(n, seed=4))
    norm = nnb.Normalization(theta=0.2, valid=True)
    x1, _ = nnb.solve_sparse_factorized(csr, b, 63, norm)
    x8, _ = nnb.solve_sparse_factorized_sharded_emulated(csr, b, 63, norm, 8)
    torch.cuda.synchronize()
    assert torch.equal(x1, x8)
    assert nnb.sparse_last_format() == "row-dictionary-stencil-tb"  # 8 slabs of 512 grid rows


def test_sparse_sharded_nccl_world1(ref):
    rp, col, val = W.laplacian_5pt(40)
    b = W.rhs(1600, seed=2)
    comm = nnb.Comm(1, 0, nnb.Comm.unique_id())
    try:
        xs, cnt = nnb.solve_sparse_factorized_sharded(comm, nnb.Csr(rp, col, val, n=1600), 1600, b, 31,
                                                      nnb.Normalization(theta=0.2, valid=True))
    finally:
        comm.close()
    xr, _, _ = ref.sparse_factorized(rp, col, val, b, 31, 0.2)
    assert cnt == 31 and np.array_equal(xs, xr.real)


def test_sparse_sharded_rejects_wide_halo():
    # a dense coupling between the first and last rows spans every slab
    n = 64
    rows, cols = np.arange(n), np.arange(n)
    dense = np.eye(n) * 4.0
    dense[0, n - 1] = dense[n - 1, 0] = -1.0
    rp = np.zeros(n + 1, np.int64)
    cl, vl = [], []
    for i in range(n):
        nz = np.nonzero(dense[i])[0]
        cl.extend(nz)
        vl.extend(dense[i, nz])
        rp[i + 1] = len(cl)
    csr = nnb.Csr(rp, np.array(cl, np.int32), np.array(vl), n=n)
    with pytest.raises(nnb.DomainError):
        nnb.solve_sparse_factorized_sharded_emulated(csr, np.ones(n), 7, nnb.Normalization(theta=0.2, valid=True), 4)


def test_sparse_plan_reuse_nccl_world1(ref):
    """The prepared slab (nnb_sparse_plan_*) serves repeated solves, bit-exact each time."""
    rp, col, val = W.laplacian_5pt(50)
    comm = nnb.Comm(1, 0, nnb.Comm.unique_id())
    plan = nnb.SparseShardedPlan(comm, nnb.Csr(rp, col, val, n=2500), 2500, k=1)
    try:
        for seed in (1, 2, 3):
            b = W.rhs(2500, seed=seed)
            x, cnt = plan.solve(b, 63, nnb.Normalization(theta=0.2, valid=True))
            xr, _, _ = ref.sparse_factorized(rp, col, val, b, 63, 0.2)
            assert cnt == 63 and np.array_equal(x, xr.real)
    finally:
        plan.close()
        comm.close()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_c4_emulated_sharded_matches_single_gpu_n8192(world):
    """SURVEY §8(c) C4 item (ii) at N=8192: the row-sharded schedule (ring all-gathers,
    K-split partial products, rank-ordered eps) over 2/4/8 virtual ranks gives the
    single-GPU X to 1e-12 relative, and the same eps history."""
    import torch

    n = 8192
    g = torch.Generator(device="cuda").manual_seed(8192)
    b = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
    a = torch.addmm(torch.eye(n, dtype=torch.float64, device="cuda"), b, b.T, alpha=1.0 / n)
    del b
    x1, r1 = nnb.nn_chain(a, None, p=2, max_iters=3)
    xs, rs = nnb.nn_chain_sharded_emulated(a, world, None, p=2, max_iters=3)
    assert rs.iters == r1.iters == 3 and rs.products == r1.products
    rel = (torch.linalg.norm(torch.as_tensor(xs, device="cuda") - x1) / torch.linalg.norm(x1)).item()
    assert rel < 1e-12, rel
    e1 = np.array([e for _, e in r1.history])
    es = np.array([e for _, e in rs.history])
    assert np.allclose(es, e1, rtol=1e-10, atol=1e-15)


def _np(x):
    import torch

    return torch.as_tensor(x).cpu().numpy() if not isinstance(x, np.ndarray) else x


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_emulated_sharded_int8_emulation_bit_identical(world):
    """The sharded int8-emulated products (column statistics gathered and combined in rank
    order, residue blocks all-gathered, G block GEMMs accumulated mod m_l, one
    reconstruction) give the single-GPU emulated chain's X bit for bit (N=4096, the FAST
    mode's int8 path; ragged blocks at world 3)."""
    import torch

    n = 4096
    g = torch.Generator(device="cuda").manual_seed(4096)
    b = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
    a = torch.addmm(torch.eye(n, dtype=torch.float64, device="cuda"), b, b.T, alpha=1.0 / n)
    del b
    x1, r1 = nnb.nn_chain(a, None, p=2, max_iters=3)
    xs, rs = nnb.nn_chain_sharded_emulated(a, world, None, p=2, max_iters=3)
    assert rs.iters == r1.iters == 3 and rs.products == r1.products
    x1, xs = _np(x1), _np(xs)
    assert np.array_equal(xs, x1), rel_frob(xs, x1)
    e1 = np.array([e for _, e in r1.history])
    es = np.array([e for _, e in rs.history])
    assert np.allclose(es, e1, rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("world", [3, 8])
def test_emulated_sharded_forced_int8_ragged(port, world):
    """NNB_ARITH_OZAKI at N=1000 (63 16-row units over 3 or 8 ranks: blocks of 336/328 and
    128/104 rows, partial 128-row tiles, K blocks that are not multiples of the 128-byte
    k-tile): bit-identical to the single-GPU emulated chain, and the oracle to 1e-10."""
    n = 1000
    a = W.gram_shifted(n, seed=3, shift=1.0)
    with nnb.ozaki_arithmetic():
        x1, r1 = nnb.nn_chain(a, None, p=3, max_iters=5)
        xs, rs = nnb.nn_chain_sharded_emulated(a, world, None, p=3, max_iters=5)
    assert np.array_equal(_np(xs), _np(x1)), rel_frob(_np(xs), _np(x1))
    if world == 3:
        xr, _, _ = port.chain(a, W.x0_transpose_norm(a), 3, 5)
        assert rel_frob(_np(xs), xr.real) < 1e-10


def test_nccl_world1_int8_emulation_matches_single_gpu():
    import torch

    n = 4096
    g = torch.Generator(device="cuda").manual_seed(7)
    b = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
    a = torch.addmm(torch.eye(n, dtype=torch.float64, device="cuda"), b, b.T, alpha=1.0 / n)
    del b
    comm = nnb.Comm(1, 0, nnb.Comm.unique_id())
    try:
        xs, rs = nnb.nn_chain_sharded(comm, a, n, None, p=2, max_iters=3)
    finally:
        comm.close()
    x1, r1 = nnb.nn_chain(a, None, p=2, max_iters=3)
    assert np.array_equal(_np(xs), _np(x1))
    assert np.allclose([e for _, e in rs.history], [e for _, e in r1.history], rtol=1e-12, atol=1e-15)


def test_emulated_sharded_int8_divergence_and_tolerance(ref):
    """The int8-emulated sharded schedule keeps the chain's contracts: a non-finite start is
    reported like the single-GPU chain's (same error class), and the tolerance stop comes at
    the reference's nest (NNB_ARITH_OZAKI at N=256, 4 virtual ranks)."""
    a = W.spd_conditioned(256, 1e3, seed=9)
    x0 = W.x0_transpose_norm(a)
    with nnb.ozaki_arithmetic():
        xs, rs = nnb.nn_chain_sharded_emulated(a, 4, x0, p=2, max_iters=60, tol=1e-12)
        bad = x0.copy()
        bad[3, 5] = np.nan
        errs = []
        for fn in (lambda: nnb.nn_chain(a, bad, p=2, max_iters=4),
                   lambda: nnb.nn_chain_sharded_emulated(a, 4, bad, p=2, max_iters=4)):
            with pytest.raises(nnb.Error) as e:
                fn()
            errs.append(type(e.value))
    xr, hr, ir, _ = ref.chain(a, x0, 2, 60, tol=1e-12)
    assert rs.iters == ir and rs.stopped_reason == "tolerance"
    assert rel_frob(_np(xs), xr.real) < 1e-10
    assert errs[0] is errs[1]


def test_sparse_sharded_temporal_blocking_nonfinite(ref):
    """A non-finite right-hand side entry in one slab: the temporal-blocked slab schedule
    reports the same factor as the single-GPU solve."""
    rp, col, val = W.laplacian_5pt(64)
    b = W.rhs(4096, seed=31)
    b[2000] = np.inf
    norm = nnb.Normalization(theta=0.2, valid=True)
    with pytest.raises(nnb.DivergenceError) as e1:
        nnb.solve_sparse_factorized(nnb.Csr(rp, col, val, n=4096), b, 63, norm)
    with pytest.raises(nnb.DivergenceError) as e4:
        nnb.solve_sparse_factorized_sharded_emulated(nnb.Csr(rp, col, val, n=4096), b, 63, norm, 4)
    assert nnb.sparse_last_format() == "row-dictionary-stencil-tb"
    assert e1.value.nest_index == e4.value.nest_index
