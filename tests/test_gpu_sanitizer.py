"""compute-sanitizer over every ABI call on small inputs (memcheck, racecheck,
synccheck on the tiny configs; the code relies on spin-waits, mbarrier rings, DSMEM
and relaxed publication). Each tool runs tests/_sanitize_child.py in its own process and must
report no error (exit status of the sanitizer and its summary line)."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
CHILD = os.path.join(HERE, "_sanitize_child.py")


def _sanitizer():
    for c in (shutil.which("compute-sanitizer"), "/usr/local/cuda/bin/compute-sanitizer"):
        if c and os.path.exists(c):
            return c
    pytest.skip("compute-sanitizer not found")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck", "initcheck"])
def test_sanitizer_clean(tool):
    cmd = [_sanitizer(), "--tool", tool, "--error-exitcode", "97", "--target-processes", "all"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    if tool == "racecheck":
        cmd += ["--racecheck-report", "all"]
    env = dict(os.environ, CUDA_MODULE_LOADING="EAGER", MEMSHARE_PDL=os.environ.get("MEMSHARE_PDL", "1"))
    r = subprocess.run(cmd + [sys.executable, CHILD], cwd=os.path.dirname(HERE), env=env, timeout=1500,
                       capture_output=True, text=True)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "ok" in r.stdout, out[-4000:]
    assert "ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards" in out, out[-4000:]
