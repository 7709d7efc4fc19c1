import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a CUDA path)")


@pytest.fixture(scope="session")
def orc():
    from oracle import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle import Ref

    if not Ref.available():
        pytest.skip("oracle/_ref not built (reference tree absent when building)")
    return Ref()


@pytest.fixture(scope="session")
def ctx():
    import torch

    import paper_2504_05638_b200 as tagc

    assert torch.cuda.is_available(), "GPU test without a GPU"
    return tagc.Context(tagc.CompressionConfig(), device=0)
