"""The device-resident small-N chain (csrc/chain_small.cu: one cooperative kernel
for the whole nn_invert loop) against the launch-per-product chain (chain.cu)
and the compiled reference.  The two device paths are selected per process by
NNB_SMALL_CHAIN_MAX, so each case runs in a child process for both settings."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import rel_frob

pytestmark = pytest.mark.gpu

nnb = pytest.importorskip("paper_2212_02406_b200")
from paper_2212_02406_b200 import workloads as W  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (n, p, max_iters, tol, order, final_residual)
CASES = [
    (1, 2, 5, 0.0, 0, 1),
    (17, 0, 4, 0.0, 0, 1),
    (64, 1, 30, 1e-12, 0, 1),
    (64, 1, 30, 1e-12, 1, 1),
    (100, 3, 12, 0.0, 0, 0),
    (256, 1, 30, 0.0, 0, 1),
    (256, 2, 40, 1e-12, 1, 1),
    (300, 3, 20, 1e-12, 0, 0),
]

CHILD = r"""
import json, sys
import numpy as np
sys.path.insert(0, %(root)r)
import paper_2212_02406_b200 as nnb
from paper_2212_02406_b200 import workloads as W
out = []
for n, p, iters, tol, order, fr in %(cases)r:
    a = W.spd_conditioned(n, 50.0, seed=n + p) if n > 1 else np.array([[4.0]])
    x, rep = nnb.nn_chain(a, None, p=p, max_iters=iters, tol=tol, order=order, final_residual=bool(fr))
    np.save("%(tmp)s/x_%%d_%%d_%%d_%%d.npy" %% (n, p, order, fr), x)
    out.append(dict(iters=rep.iters, products=rep.products, stopped=rep.stopped_reason,
                    eps=[e for _, e in rep.history]))
print(json.dumps(out))
"""


def _run(tmp, small_max):
    sub = os.path.join(tmp, str(small_max))
    os.makedirs(sub, exist_ok=True)
    env = dict(os.environ, NNB_DEBUG="1", NNB_SMALL_CHAIN_MAX=str(small_max))
    code = CHILD % dict(root=ROOT, cases=CASES, tmp=sub)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return sub, json.loads(r.stdout.strip().splitlines()[-1])


def test_small_chain_matches_launch_chain(tmp_path):
    dir_small, small = _run(str(tmp_path), 512)
    dir_big, big = _run(str(tmp_path), 0)
    for case, s, b in zip(CASES, small, big):
        n, p, _, _, order, fr = case
        assert (s["iters"], s["products"], s["stopped"]) == (b["iters"], b["products"], b["stopped"]), case
        es, eb = np.array(s["eps"]), np.array(b["eps"])
        assert es.shape == eb.shape, case
        # 1e-10 relative, plus the absolute rounding noise of an ε computed from N² terms;
        # the floor region (both below 1e-12) compares only as "both below"
        floor = (es < 1e-12) & (eb < 1e-12)
        assert np.all(floor | (np.abs(es - eb) <= 1e-10 * eb + 1e-15)), (case, np.c_[es, eb])
        name = "x_%d_%d_%d_%d.npy" % (n, p, order, fr)
        xs, xb = np.load(os.path.join(dir_small, name)), np.load(os.path.join(dir_big, name))
        assert rel_frob(xs, xb) < 1e-12, case


def test_small_chain_c1_vs_reference_and_divergence(ref):
    """Config 0 through the small kernel (the default for N <= 384) against the
    reference, and a start that blows up mid-chain reports the reference's nest."""
    a = W.gram_shifted(256, seed=2212, shift=0.5)
    x0 = W.x0_transpose_norm(a)
    xr, hr, ir, _ = ref.chain(a, x0, 1, 30)
    x, rep = nnb.nn_chain(a, x0, p=1, max_iters=30)
    assert rep.iters == ir == 30 and rel_frob(x, xr.real) < 1e-10
    big = 1e150 * np.eye(64)
    with pytest.raises(nnb.DivergenceError) as e:
        nnb.nn_chain(np.eye(64), big, p=2, max_iters=10)
    assert e.value.nest_index >= 1
