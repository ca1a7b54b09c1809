import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; run with -m gpu")
    config.addinivalue_line("markers", "reference: needs the read-only reference checkout (/root/reference)")


def pytest_collection_modifyitems(config, items):
    have_ref = REFERENCE_SRC.exists()
    skip_ref = pytest.mark.skip(reason="reference checkout not present (GPU box)")
    for item in items:
        if "reference" in item.keywords and not have_ref:
            item.add_marker(skip_ref)


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test collected without a CUDA device (run -m gpu on a B200)")
    from paper_2509_19836_b200 import _native

    _native.load()  # fail loudly if the kernel library is missing
    return torch.device("cuda:0")
