import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def vtc():
    import paper_2604_09558_b200 as m
    return m


@pytest.fixture(scope="session")
def ref():
    import ref as r
    if not r.available():
        pytest.skip("oracle/_ref not built (make -C oracle)")
    return r


@pytest.fixture(scope="session")
def oracle():
    import vtc_oracle as o
    return o
