"""The shared-memory-resident Householder kernel (k_lsq_sm) on every shape it
accepts.  By default the dispatcher uses it for complex shapes with r+1 >= 16
(config 4); SAS_LSQ_SM=1 (read once per process) routes every fitting real
shape to it as well, so the whole dispatch suite -- random weighted affine
problems with repeated rows against the CPU oracle, rank-deficient and
non-finite cases -- runs again in a child process with that setting."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


def test_dispatch_suite_with_shared_memory_kernel_forced():
    env = dict(os.environ, SAS_LSQ_SM="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        str(ROOT / "tests" / "test_gpu_dispatch.py")],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
