import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device; run with -m gpu")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the product library and the oracle once (no-ops when up to date)."""
    from oracle import oracle
    from paper_2601_19911_b200.csrc import build

    build.build()
    oracle.build()


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device in this container")
    return torch.device("cuda", 0)


@pytest.fixture(scope="session")
def b200(cuda):
    from paper_2601_19911_b200 import B200Device

    dev = B200Device()
    yield dev
    dev.close()
