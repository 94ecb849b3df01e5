import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
FIXTURES = ["single_bus", "two_bus", "three_bus_transformer", "four_bus_delta", "two_bus_delta"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (large synthetic feeders)")


def fixture_path(name: str) -> str:
    return os.path.join(GOLDEN, "fixtures", name + ".json")


@pytest.fixture(scope="session", autouse=True)
def _built():
    # build the in-tree libraries once (no-op when up to date)
    from paper_2501_08293_b200 import build
    build.build_host()
    build.build_oracle()
    yield


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
