import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (large configs)")
    # make sure libmvn.so (and the C oracle) exist and are not older than their sources: nvcc
    # cross-compiles for sm_100a without a GPU, so this works on the CPU box too
    try:
        from paper_2405_14892_b200 import _build
        _build.build()
        import oracle
        oracle.build()
    except Exception as e:  # pragma: no cover - reported by the tests that need the library
        sys.stderr.write(f"conftest: library build skipped: {e}\n")


@pytest.fixture(scope="session")
def cuda_device():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")
