import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libdm_moe.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    major, minor = torch.cuda.get_device_capability()
    if major != 10:
        pytest.skip(f"needs sm_100 (got sm_{major}{minor})")
    from paper_2605_11005_b200 import build

    build.build()
    return torch.device("cuda:0")


@pytest.fixture(scope="session")
def golden_dir():
    return ROOT / "tests" / "golden"
