import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: large sizes, minutes on the GPU box")


def _have_cuda() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


HAVE_CUDA = _have_cuda()


def pytest_collection_modifyitems(config, items):
    if HAVE_CUDA:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def oracle():
    """The C restatement of the reference (the parity checker)."""
    from oracle import binding

    return binding.get("restatement")


@pytest.fixture(scope="session")
def ref():
    """The compiled reference library (oracle/_ref), when it was built."""
    from oracle import binding

    if not binding.available("reference"):
        pytest.skip("oracle/_ref not built")
    return binding.get("reference")


@pytest.fixture(scope="session")
def mg():
    import paper_2401_05994_b200 as m

    if HAVE_CUDA:
        from paper_2401_05994_b200 import _lib

        _lib.lib()
    return m
