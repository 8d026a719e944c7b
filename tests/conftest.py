import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


@pytest.fixture(scope="session")
def cuda_lib():
    """The product C-ABI library on cuda:0 (GPU tests only)."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but torch.cuda.is_available() is False")
    import paper_2605_15565_b200 as rl
    rl.load()
    # RL_TEST_DEV_OPTS="key=value,...": development options for this process (test_gpu_kernels.py)
    for kv in filter(None, os.environ.get("RL_TEST_DEV_OPTS", "").split(",")):
        k, v = kv.split("=")
        rl.dev_set_option(int(k), int(v))
    return rl
