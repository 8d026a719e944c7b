"""The non-default kernels, selected per process through the library's development options
(include/rl_policy_dev.h, rl_dev_set_option; the test harness applies RL_TEST_DEV_OPTS in
conftest.py — the library itself never reads the environment), against the same oracle parity
tests as the default ones."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("opts,select", [
    ("0=1", "tiny or ragged or knobs or unit_scale or masked or extreme or sum_to_zero or objective"),  # two-pass loss
    ("1=1", "vocab_parallel"),  # NCCL vocab-parallel path
    ("3=1", "vocab_parallel"),  # L2 re-read ring kernel instead of the register-cache kernel
])
def test_alternate_kernels(opts, select):
    env = dict(os.environ, RL_TEST_DEV_OPTS=opts)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-k", select],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
