import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device; run with -m gpu")


@pytest.fixture(scope="session")
def oracle():
    from oracle import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle import Reference

    if not Reference.available():
        pytest.skip("reference library (oracle/_ref) not built here")
    return Reference()


@pytest.fixture(scope="session")
def rs():
    """The product package, on a GPU; fails (not skips) if the library is
    missing so a silent fallback can never pass."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2107_01391_b200 as rs

    rs._lib.load()
    return rs


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    path = os.path.join(ROOT, "tests", "golden", "ref_vectors.npz")
    return dict(np.load(path, allow_pickle=False))
