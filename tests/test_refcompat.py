"""The reference's own hot-path unit tests (proj/tests/test_sketches.cpp,
test_core_linalg.cpp, test_preconditioning.cpp, test_solvers.cpp,
test_sketch_stats.cpp, test_distsim.cpp), compiled
UNMODIFIED with the Catch2-compatible shim (tests/refcompat/) against
  * the reference headers alone (CPU): checks the shim reproduces the
    reference's own verdicts;
  * the B200 drop-in headers (include/sketchlsq_b200) + libslq_b200.so (GPU):
    the drop-in passes the reference's tests.
Built by tests/refcompat/Makefile (needs /root/reference; __graft_entry__.build)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "tests", "refcompat", "_build")
TESTS = ["test_sketches", "test_core_linalg", "test_preconditioning", "test_solvers", "test_sketch_stats",
         "test_distsim"]
# a wall-clock assertion of the reference (t(zeta=24) / t(zeta=8) in [2, 4.5] on
# the CPU generator, test_sketch_stats.cpp:196-209): it depends on the host it
# runs on (the reference itself measures 4.9 in this container), so its
# verdict is reported but not required
TIMING_CASES = {"generation cost scales with zeta not d"}


def _bin(name):
    p = os.path.join(BUILD, name)
    if not os.path.exists(p):
        pytest.skip(f"{name} not built (make -C tests/refcompat needs /root/reference)")
    return p


def _run(path):
    out = subprocess.run([path], capture_output=True, text=True, timeout=1200)
    m = re.search(r"test cases: (\d+) passed, (\d+) failed", out.stdout)
    assert m, out.stdout[-2000:] + out.stderr[-2000:]
    failed = {l[6:].strip() for l in out.stdout.splitlines() if l.startswith("FAIL  ")}
    return int(m.group(1)), failed - TIMING_CASES, out


@pytest.mark.parametrize("t", TESTS)
def test_shim_reproduces_reference_verdicts(t):
    passed, failed, out = _run(_bin(f"{t}_ref"))
    assert not failed and passed > 0, out.stderr[-3000:]


@pytest.mark.parametrize("t", TESTS)
def test_dropin_binary_links_the_b200_library(t):
    p = _bin(f"{t}_dropin")
    syms = subprocess.run(["nm", "-D", p], capture_output=True, text=True).stdout
    assert re.search(r"\bU slq_", syms), "drop-in test binary does not call the C-ABI"


@pytest.mark.gpu
@pytest.mark.parametrize("t", TESTS)
def test_reference_tests_pass_on_the_dropin(t):
    _, failed_ref, out_ref = _run(_bin(f"{t}_ref"))
    passed, failed, out = _run(_bin(f"{t}_dropin"))
    assert not failed, out.stdout[-3000:] + out.stderr[-4000:]
    cases = lambda o: {l[6:].strip() for l in o.stdout.splitlines() if l[:6] in ("PASS  ", "FAIL  ")}
    assert cases(out) == cases(out_ref)
