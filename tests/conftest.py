import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(autouse=True)
def _checked_build_status(request):
    """DT_CHECKED_RUN=1 (tools/checked_build.sh, on the GPU box, with libdifftrans built with
    -DDT_CHECKED=1): after every GPU test, every in-kernel bounds check must have held."""
    yield
    if os.environ.get("DT_CHECKED_RUN") != "1" or "gpu" not in request.keywords:
        return
    from paper_2603_00413_b200 import _native
    st = _native.check_status()
    assert all(v == 0 for v in st.values()), f"in-kernel bounds check failed (source lines): {st}"
