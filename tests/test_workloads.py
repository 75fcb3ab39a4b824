import numpy as np

from paper_2212_02406_b200 import workloads as W


def test_laplacian_structure():
    g = 9
    rp, col, val = W.laplacian_5pt(g)
    n = g * g
    assert rp[-1] == 5 * n - 4 * g == col.size == val.size
    assert rp.dtype == np.int64 and col.dtype == np.int32
    for r in range(n):  # canonical CSR: strictly increasing columns, diag 5
        cs = col[rp[r]:rp[r + 1]]
        assert np.all(np.diff(cs) > 0) and r in cs
        assert val[rp[r] + list(cs).index(r)] == 5.0


def test_gram_and_spd():
    a = W.gram_shifted(64, 3, 0.5)
    assert np.array_equal(a, a.T) and np.linalg.eigvalsh(a).min() >= 0.5 - 1e-12
    s = W.spd_conditioned(64, 1e3, 4)
    ev = np.linalg.eigvalsh(s)
    assert abs(ev.max() / ev.min() - 1e3) < 1e-6 * 1e3


def test_mimo_gram():
    a = W.mimo_gram_host(8, 1)
    assert a.shape == (8, 16, 16)
    assert np.array_equal(a, np.conj(np.transpose(a, (0, 2, 1))))  # exactly Hermitian
    assert np.all(np.linalg.eigvalsh(a) >= 0.1 - 1e-12)
    # E[diag] = 1 + sigma^2 for CN(0, 1/128) entries over 128 antennas
    assert abs(np.mean(np.real(np.diagonal(a, axis1=1, axis2=2))) - 1.1) < 0.1


def test_x0_builders_contract():
    a = W.gram_shifted(32, 5, 0.5)
    x0 = W.x0_transpose_norm(a)
    # ||I - X0 A||_2 < 1 for SPD A (the NN contraction precondition)
    assert np.linalg.norm(np.eye(32) - x0 @ a, 2) < 1
