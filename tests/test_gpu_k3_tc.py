"""The opt-in tensor-core K3 (OZK_K3_TC=1, csrc/k3_tc.cu: C1 = sum s1_i u_i as a
u8 x u8 tcgen05 MMA against the base-256 digits of the FP64 s1 table) is held to
the same bar as the production kernel: the randomised parity sweep, run in a
child process because the library reads the switch once per process, in both
tile shapes (8 and 4 rows per thread)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("rows", ["8", "4"])
def test_k3_tc_random_sweep(rows):
    env = dict(os.environ, OZK_K3_TC="1", OZK_K3_TC_ROWS=rows)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_random.py")],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
