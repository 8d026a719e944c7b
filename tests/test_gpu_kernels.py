"""The non-default kernels (selected per process with RL_LOSS_KERNEL / RL_LOGPROB_KERNEL / RL_VP_KERNEL / RL_DELTA_ALGO / RL_VP_FUSED / RL_VP2_WPR, latched
on first use) against the same oracle parity tests as the default ones."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("var,kernel,select", [
    ("RL_LOSS_KERNEL", "cluster", "tiny or ragged or knobs or unit_scale or masked or extreme or sum_to_zero or objective"),
    ("RL_LOSS_KERNEL", "two_pass", "tiny or ragged or knobs or unit_scale or masked or extreme or sum_to_zero or objective"),
    ("RL_LOGPROB_KERNEL", "block", "token_logprob"),
    ("RL_VP_KERNEL", "block", "vocab_parallel"),
    ("RL_DELTA_ALGO", "onepass", "delta"),
    ("RL_VP_FUSED", "smem", "vocab_parallel"),
    ("RL_VP2_WPR", "4", "vocab_parallel"),
    ("RL_VP2_WPR", "16", "vocab_parallel"),
])
def test_alternate_kernels(var, kernel, select):
    env = dict(os.environ, **{var: kernel})
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-k", select],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
