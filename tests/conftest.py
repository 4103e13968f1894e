import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 CUDA devices")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the in-tree native libraries once (no-op when up to date)."""
    from paper_2106_10207_b200 import _build

    if os.environ.get("SP_SKIP_BUILD") != "1" and os.path.exists(_build.NVCC):
        _build.build_all()
        from oracle import build_ref

        build_ref.build()  # no-op without /root/reference (the GPU box uses the prebuilt .so)
    yield
