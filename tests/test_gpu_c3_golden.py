"""BASELINE config 2 at its stated size against the reference.

tests/golden/c3_n4096.npz comes from tests/golden/make_golden_c3.py: the reference's
loop (proj/src/solver.cpp:138-159, explicit X0) run offline on nn::random_spd(4096, 1e3, 3)
through the C restatement that test_oracle_pins.py pins bit for bit to the reference (and,
in the fixture, whose first N=4096 nest was checked bit for bit against oracle/_ref).
North_star gate: identical nest counts to eps < 1e-12 for p = 1, 2, 3; eps within 1e-6
rel + 1e-13 (floor entries as "both < 1e-12"); the 64x64 seeded sample of X within 1e-10
relative Frobenius — on both product paths (int8 emulation and DMMA) and both orders."""
import hashlib
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

nnb = pytest.importorskip("paper_2212_02406_b200")
from paper_2212_02406_b200 import workloads as W  # noqa: E402

G = Path(__file__).resolve().parent / "golden" / "c3_n4096.npz"


@pytest.fixture(scope="module")
def c3():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device")
    g = dict(np.load(G))
    a = nnb.random_spd(4096, 1e3, 3)  # the reference's generator, on the device
    assert hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest() == str(g["a_sha256"])
    x0 = W.x0_transpose_norm(a)
    assert hashlib.sha256(np.ascontiguousarray(x0).tobytes()).hexdigest() == str(g["x0_sha256"])
    return g, torch.from_numpy(a).cuda(), torch.from_numpy(x0).cuda()


def eps_close(a, b):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, (a.shape, b.shape)
    floor = (a < 1e-12) & (b < 1e-12)
    ok = floor | (np.abs(a - b) <= 1e-6 * b + 1e-13)
    assert ok.all(), np.c_[a, b][~ok]


def test_fixture_pinned_to_reference():
    g = dict(np.load(G))
    assert bool(g["ref_first_nest_bitexact"])
    assert (int(g["iters_p1"]), int(g["iters_p2"]), int(g["iters_p3"])) == (32, 21, 16)


@pytest.mark.parametrize("mode", ["fast", "dmma"])
@pytest.mark.parametrize("order", ["northstar", "reference"])
@pytest.mark.parametrize("p", [1, 2, 3])
def test_c3_full_size_matches_reference(c3, p, order, mode):
    g, a, x0 = c3
    ord_ = nnb.ORDER_NORTHSTAR if order == "northstar" else nnb.ORDER_REFERENCE
    ctx = nnb.arithmetic(nnb.ARITH_FAST if mode == "fast" else nnb.ARITH_DMMA)
    with ctx:
        x, rep = nnb.nn_chain(a, x0, p=p, max_iters=80, tol=1e-12, order=ord_)
    assert rep.stopped_reason == "tolerance"
    assert rep.iters == int(g[f"iters_p{p}"])
    eps_close([e for _, e in rep.history], g[f"eps_p{p}"])
    rows, cols = g["rows"], g["cols"]
    xs = x.cpu().numpy()[np.ix_(rows, cols)]
    ref = g[f"xs_p{p}"]
    assert np.linalg.norm(xs - ref) / np.linalg.norm(ref) < 1e-10
    assert abs(float(x.norm()) - float(g[f"xfrob_p{p}"])) / float(g[f"xfrob_p{p}"]) < 1e-10
