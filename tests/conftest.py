import os
import sys

import pytest

# 28 concurrent launch-group streams need 32 hardware queues (read by CUDA at
# context creation; the library itself never sets it -- engine.cpp Context())
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def lfgpu():
    from paper_2509_10712_b200 import lfgpu as L
    return L


@pytest.fixture(scope="session")
def oracle():
    import lf_oracle
    return lf_oracle
