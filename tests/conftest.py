import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built extension")
    config.addinivalue_line("markers", "slow: full-size configs")


@pytest.fixture(scope="session")
def oracle():
    from oracle.cpu import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.cpu import Reference

    if not Reference.available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Reference()


@pytest.fixture(scope="session")
def ctx():
    from paper_2504_14338_b200 import api

    c = api.DeviceContext(device=int(os.environ.get("DOPINF_DEVICE", "0")))
    yield c
    c.close()


def rel_frob(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
