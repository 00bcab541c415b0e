"""The C++ drop-in header (include/sketchlsq_b200/sketchlsq.hpp) driving the B200:
examples/dropin_solve.cpp is the reference's serial solve sequence
(test_solvers.cpp:25-37) compiled against the drop-in and linked to
libslq_b200.so (built by __graft_entry__.build())."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_dropin_example_runs_on_gpu():
    exe = os.path.join(ROOT, "examples", "dropin_solve")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", os.path.join(ROOT, "examples")], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "termination=" in out.stdout and "InvalidSparsity ok" in out.stdout
    assert "hbm iterations=" in out.stdout and "InvalidDistortion ok" in out.stdout
