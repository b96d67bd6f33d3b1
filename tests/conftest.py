"""pytest configuration: the `gpu` marker and shared helpers.

`-m "not gpu"` runs here (no GPU): oracle pinning, host planning, ABI exports.
`-m gpu` runs on a B200 through gpurun: parity of the CUDA path vs the oracle.
"""
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run through gpurun)")


@pytest.fixture(scope="session")
def orc():
    from oracle import pyoracle
    return pyoracle.orc()


@pytest.fixture(scope="session")
def ref():
    from oracle import pyoracle
    r = pyoracle.ref()
    if r is None:
        pytest.skip("oracle/_ref not built (no /root/reference when it was built)")
    return r


@pytest.fixture(scope="session")
def golden():
    import numpy as np
    d = ROOT / "tests" / "golden"
    return {p.stem: dict(np.load(p, allow_pickle=False)) for p in d.glob("*.npz")}
