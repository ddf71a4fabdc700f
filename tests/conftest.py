import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))
sys.path.insert(0, str(ROOT / "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "multigpu: needs >= 2 CUDA devices")
    config.addinivalue_line("markers", "slow: long-running")


def _device_count() -> int:
    try:
        from paper_1802_06949_b200 import device_count
        return device_count()
    except Exception:
        return 0


@pytest.fixture(scope="session")
def ngpus() -> int:
    return _device_count()


@pytest.fixture(scope="session")
def gpu(ngpus):
    if ngpus < 1:
        pytest.fail("test marked gpu but no CUDA device is visible")
    import torch
    torch.cuda.init()
    return 0


@pytest.fixture(scope="session")
def two_gpus(ngpus):
    if ngpus < 2:
        pytest.skip("needs >= 2 GPUs (gpurun --gpus 2)")
    return ngpus
