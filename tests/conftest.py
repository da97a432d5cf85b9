import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libvrg.so")
    config.addinivalue_line("markers", "slow: long-running CPU oracle comparison")


@pytest.fixture(scope="session")
def ctx():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1604_02153_b200 import api

    c = api.Context(0)
    yield c
    c.sync()


@pytest.fixture(scope="session")
def ref():
    """The compiled unmodified reference (oracle/_ref), built by `make -C oracle`."""
    from oracle import ref as R

    if not R.available():
        pytest.skip("oracle/_ref/libveloreg_ref.so not built")
    return R
