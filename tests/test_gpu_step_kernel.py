"""The single-sequence step kernel (csrc/step.cu, opt-in with TS_STEP=1; the
library reads the switch at load time) against the oracle: the decode
parity tests of test_gpu_parity.py and the 128K rotating-stream test of
test_gpu_configs.py, in a subprocess with the switch on."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_step_kernel_decode_parity():
    env = dict(os.environ, TS_STEP="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        "tests/test_gpu_parity.py", "tests/test_gpu_configs.py", "-k",
                        "decode or config2 or zero"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
