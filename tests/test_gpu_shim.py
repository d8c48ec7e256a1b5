"""The C++ drop-in shim (include/dpd_b200.hpp) driving the B200 engine."""
import os
import subprocess

import pytest

from test_abi import build_shim_example

pytestmark = pytest.mark.gpu


def test_shim_example_runs(tmp_path):
    exe = build_shim_example(str(tmp_path))
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120,
                       env=dict(os.environ, LD_LIBRARY_PATH=os.path.dirname(exe)))
    assert r.returncode == 0, r.stdout + r.stderr
    assert "shim ok" in r.stdout
    assert "fastlog(2^31)=-0.69314718055994529" in r.stdout
