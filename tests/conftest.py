import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libtofr_b200.so")


@pytest.fixture(scope="session")
def renderer():
    from paper_2605_11536_b200.api import Renderer
    return Renderer(0)


@pytest.fixture(scope="session")
def ref():
    from oracle import ref as R
    if not R.available():
        R.build_if_possible()
    if not R.available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return R
