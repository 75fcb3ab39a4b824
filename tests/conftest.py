import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests of the CUDA path")


def rel_frob(a, b) -> float:
    """||a - b||_F / ||b||_F (absolute when b is zero), like the reference's rel_frob_diff
    (proj/tests/support/oracles.hpp:35-36)."""
    a = np.asarray(a)
    b = np.asarray(b)
    nb = np.linalg.norm(b)
    d = np.linalg.norm(a - b)
    return d / nb if nb > 0 else d


@pytest.fixture(scope="session")
def port():
    import os

    from oracle import Port

    p = Port()
    p.set_threads(os.cpu_count() or 1)  # row-partitioned like the reference; bit-identical for any count
    return p


@pytest.fixture(scope="session")
def ref():
    from oracle import Reference, have_ref

    if not have_ref():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Reference()


def golden(name: str):
    return dict(np.load(GOLDEN / name))
