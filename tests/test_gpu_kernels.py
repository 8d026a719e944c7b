"""The non-default fused-loss kernels (selected per process with RL_LOSS_KERNEL, latched on
first use) against the same oracle parity tests as the default single-visit kernel."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("kernel", ["cluster", "two_pass"])
def test_alternate_loss_kernels(kernel):
    env = dict(os.environ, RL_LOSS_KERNEL=kernel)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_parity.py"),
                        "-k", "tiny or ragged or knobs or unit_scale or masked or extreme or sum_to_zero"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
