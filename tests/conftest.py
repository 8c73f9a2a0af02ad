import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs the product library)")
    config.addinivalue_line("markers", "slow: long-running")


def _gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def pytest_collection_modifyitems(config, items):
    if _gpu_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


IMPLS = [pytest.param("product", marks=pytest.mark.gpu), "oracle", "reference"]


@pytest.fixture(params=IMPLS)
def impl(request):
    """Backend under test: the B200 product, the CPU restatement, or the compiled reference."""
    import support as S

    if request.param == "product":
        return S.product_backend()
    b = S.oracle_backend() if request.param == "oracle" else S.ref_backend()
    if b is None:
        pytest.skip(f"{request.param} library not built")
    return b
