"""CPU tests of the boundary: the C-ABI library loads, exports every symbol
include/slq_b200.h declares, and its host-only logic (partition_rows, error
mapping) matches the oracle.  No kernels run here (no GPU in this container)."""
import os
import re

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lib():
    from paper_2506_03070_b200 import _capi

    return _capi


def test_library_exports_header_symbols():
    capi = _lib()
    with open(os.path.join(ROOT, "include", "slq_b200.h")) as f:
        hdr = f.read()
    names = set(re.findall(r"^\s*(?:int|int64_t|const char\*|void)\s+(slq_\w+)\s*\(", hdr, re.M))
    assert len(names) >= 25
    for nme in sorted(names):
        assert hasattr(capi.lib, nme), nme
    assert set(capi.EXPORTED) == names


def test_partition_rows_matches_reference():
    import paper_2506_03070_b200 as slq

    C = oracle.C()
    for m, p in [(333, 1), (333, 2), (333, 4), (333, 8), (4_000_000, 8), (1 << 20, 3), (7, 7)]:
        assert slq.partition_rows(m, p).boundaries == C.partition_rows(m, p).tolist()
    with pytest.raises(slq.InvalidDims):
        slq.partition_rows(3, 4)
    with pytest.raises(slq.InvalidDims):
        slq.partition_rows(3, 0)


def test_no_gpu_fails_loudly():
    import torch

    import paper_2506_03070_b200 as slq

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(slq.CudaError):
        slq.generate_sparse_sign(16, 6, 4, 7)


def test_solve_options_defaults_match_reference():
    import paper_2506_03070_b200 as slq
    from paper_2506_03070_b200 import _capi
    import ctypes as ct

    o = _capi.SolveOpts()
    _capi.lib.slq_solve_opts_default(ct.byref(o))
    assert o.eps == 1e-10 and o.maxit == 100  # lsqr.hpp:15-16
    so = slq.SolveOptions()
    assert so.eps == 1e-10 and so.maxit == 100


def test_report_json_shape():
    import paper_2506_03070_b200 as slq

    r = slq.SolveReport(residual_estimate=[1.0, 0.5], iterations=2, termination=slq.Termination.MaxIter,
                        sync_count=3, init_reductions=1)
    j = r.to_json()
    assert j["termination"] == "maxiter" and j["reductions_per_iteration"] == 1.0
    assert "iterates_error" not in j
