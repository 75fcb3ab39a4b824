"""The C-ABI library loads and exports every entry point include/nnb.h declares
(CPU-safe: no compute calls are made without a GPU)."""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared():
    text = (ROOT / "include" / "nnb.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(nnb_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    names = declared()
    assert "nnb_nn_chain_d" in names and "nnb_sparse_factorized_d" in names and len(names) >= 24


def test_library_exports_all_declared_symbols():
    from paper_2212_02406_b200 import LIB_PATH, exported_symbols

    if not LIB_PATH.exists():
        pytest.fail("libnnb.so not built: run `make` (python -c 'import __graft_entry__ as g; g.build()')")
    lib = ctypes.CDLL(str(LIB_PATH))
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(exported_symbols()) == set(declared())


def test_abi_version_and_no_cpu_fallback():
    import paper_2212_02406_b200 as nnb

    L = nnb.lib()
    assert L.nnb_abi_version() == 1
    if L.nnb_device_count() == 0:
        # without a GPU a compute entry point refuses instead of computing on the host
        import numpy as np

        a = np.eye(4)
        with pytest.raises(nnb.DeviceError):
            nnb.matmul(a, a)


def test_gaussian_stream_matches_reference(ref):
    """nnb_gaussian_stream (host) reproduces nn::GaussianStream bit for bit."""
    import paper_2212_02406_b200 as nnb

    for seed, count in ((42, 7), (1, 1), (99, 10001)):
        assert np.array_equal(nnb.gaussian_stream(seed, count), ref.gaussian(seed, count))
