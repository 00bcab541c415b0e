"""Out-of-bounds device writes into the library's scratch buffers: the whole
hot path (K1, K2 gathers incl. K2d's stage refill, K3 cluster panel / updates /
TSQR, K4 rings incl. the wide-row pass, K5, the sparse one- and two-pass
operators and the transposed-copy build, the gradient family) runs with
SLQ_GUARD=1, which surrounds every DevBuf allocation with 64 KB guard bands;
every band must be intact afterwards (slq_debug_check_guards).  A stand-in for
compute-sanitizer memcheck, which is closed on this GPU pool."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_guard_bands_intact_after_hot_path_workload():
    env = dict(os.environ, SLQ_GUARD="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_workload.py")], env=env,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("guards_corrupted=")]
    assert line, out.stdout[-2000:]
    assert line[-1] == "guards_corrupted=0", out.stdout[-2000:] + out.stderr[-2000:]


def test_guard_mechanism_detects_a_planted_overrun():
    code = ("import ctypes as ct, paper_2506_03070_b200 as slq; d = ct.c_int(-1); "
            "assert slq._capi.lib.slq_debug_guard_selftest(ct.byref(d)) == 0; print('detected', d.value)")
    env = dict(os.environ, SLQ_GUARD="1", PYTHONPATH=ROOT)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    assert "detected 1" in out.stdout, out.stdout + out.stderr
