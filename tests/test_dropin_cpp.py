"""The C++ drop-in surface (namespace nn, paper_2212_02406_b200/dropin) driven by
tests/cpp/test_dropin.cpp — the reference's hot-path unit tests restated."""
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "build" / "test_dropin"


def _bin():
    if not BIN.exists():
        subprocess.run(["make", "-s", "-C", str(ROOT), "dropin"], check=True)
    return str(BIN)


def test_dropin_host_checks_and_gaussian_stream(ref):
    out = subprocess.run([_bin(), "--host"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    vals = [float(v) for v in re.search(r"gaussian42:(.*)", out.stdout).group(1).split()]
    # nn::GaussianStream of the drop-in reproduces the reference's stream bit-for-bit
    assert np.array_equal(np.array(vals), ref.gaussian(42, 6))


@pytest.mark.gpu
def test_dropin_device_suite():
    out = subprocess.run([_bin()], capture_output=True, text=True, timeout=900)
    print(out.stdout[-3000:])
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
    assert ", 0 failures" in out.stdout
