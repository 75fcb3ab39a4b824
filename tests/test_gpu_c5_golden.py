"""BASELINE config 4 at its stated size against the reference, bit for bit (VERDICT r01
item 1): the 4096^2 Laplacian + I solve (gamma = 63, theta = 0.2) on the GPU -- single
device, and the row-slab schedule emulated with 8 ranks -- hashes to the reference's x
(tests/golden/c5_n4096.npz, made by oracle/_ref through make_golden_c5.py)."""
import hashlib
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

nnb = pytest.importorskip("paper_2212_02406_b200")
from paper_2212_02406_b200 import workloads as W  # noqa: E402

G = Path(__file__).resolve().parent / "golden" / "c5_n4096.npz"


@pytest.fixture(scope="module")
def c5():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device")
    g = dict(np.load(G))
    rp, col, val = W.laplacian_5pt(4096)
    b = W.rhs(4096 * 4096, seed=7)
    assert hashlib.sha256(np.ascontiguousarray(b).tobytes()).hexdigest() == str(g["b_sha256"])
    dev = lambda v: torch.from_numpy(v).cuda()
    return g, nnb.Csr(dev(rp), dev(col), dev(val), n=4096 * 4096, nnz=col.size), dev(b)


def check(g, x):
    xh = np.ascontiguousarray(x.cpu().numpy())
    assert np.array_equal(xh[g["idx"]], g["x_sample"])
    assert hashlib.sha256(xh.tobytes()).hexdigest() == str(g["x_sha256"])


def test_c5_single_gpu_bit_exact(c5):
    g, csr, b = c5
    x, cnt = nnb.solve_sparse_factorized(csr, b, 63, nnb.Normalization(theta=0.2, valid=True))
    assert cnt == int(g["spmv"]) == 63
    check(g, x)


def test_c5_row_slabs_emulated_8_ranks_bit_exact(c5):
    g, csr, b = c5
    x, cnt = nnb.solve_sparse_factorized_sharded_emulated(csr, b, 63, nnb.Normalization(theta=0.2, valid=True), 8)
    assert cnt == 63
    check(g, x)
