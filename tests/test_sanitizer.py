"""compute-sanitizer over every kernel variant (memcheck, racecheck, synccheck, initcheck)."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck", "initcheck"])
def test_compute_sanitizer_clean(tool):
    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(exe):
        pytest.skip("compute-sanitizer not found")
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cmd = [exe, "--tool", tool, "--error-exitcode", "97"]
    r = subprocess.run(cmd + [sys.executable, os.path.join(HERE, "sanitizer_driver.py")],
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
    assert "sanitizer driver ok" in r.stdout
