"""Every kernel variant under the bounds-checked build (libdsi_sim_checked.so, -DDSI_BOUNDS_CHECK):
each computed index of the kernels' shared-memory tables, run slots, histograms and records is
checked (DSI_CHECK traps on the first violation).  The substitute for compute-sanitizer memcheck
where the GPU pool has the sanitizer closed (tests/test_sanitizer.py skips there)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def test_every_kernel_variant_within_bounds():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, DSI_SIM_LIB="checked")
    r = subprocess.run([sys.executable, os.path.join(HERE, "sanitizer_driver.py")], capture_output=True,
                       text=True, timeout=900, env=env)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
    assert "sanitizer driver ok" in r.stdout
    assert "DSI_CHECK failed" not in r.stdout + r.stderr
