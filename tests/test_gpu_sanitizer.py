"""compute-sanitizer memcheck on small invocations of the device paths (profiles/r01_sanitizer.md
has the full racecheck / synccheck matrix)."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
CS = "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.skipif(not os.path.exists(CS), reason="compute-sanitizer not installed")
@pytest.mark.parametrize("tool,case", [("memcheck", "apply_fast"), ("memcheck", "solve_persistent"),
                                       ("racecheck", "iteration_kernels"), ("memcheck", "solve_graph"),
                                       ("memcheck", "ic0"), ("memcheck", "io")])
def test_sanitizer_clean(tool, case):
    r = subprocess.run([CS, "--tool", tool, "--error-exitcode", "9", sys.executable,
                        os.path.join(ROOT, "tools", "sanitize_driver.py"), "--only", case],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert f"ok {case}" in r.stdout
