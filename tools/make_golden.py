"""Generate tests/golden/ fixtures from the compiled REFERENCE (oracle/_ref).

Run here (where /root/reference exists):  python tools/make_golden.py
The fixtures are small .npz files; the GPU box and the CPU test suite read
them without needing /root/reference.  Each case names the reference entry
point that produced it (see oracle/ref_shim.cpp for the file:line of each).
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")

# (d, m, zeta, seed, col_begin): forced structure, duplicate-heavy, zeta=1,
# non power-of-two zeta, zeta > 32 (generic path), global column window.
SKETCH_CASES = [
    (16, 6, 4, 7, 0),        # SURVEY Appendix A KAT
    (4, 3, 4, 1, 0),         # zeta == d forces all rows (test_sketches.cpp:10-15)
    (4, 2, 4, 9, 0),         # forced structure (test_sketches.cpp:55-66)
    (400, 64, 8, 3, 0),      # duplicate path (Appendix A: column 2)
    (16, 200, 8, 5, 0),      # duplicate-heavy: zeta^2/d = 4
    (10, 300, 9, 21, 0),     # zeta ~ d (coupon collecting), non-power-of-two
    (96, 333, 5, 271828, 0), # test_distsim.cpp:136-149 instance
    (64, 100, 8, 1234, 0),   # test_sketches.cpp:68-77
    (1000, 257, 1, 17, 0),   # zeta = 1 never dedupes
    (2000, 100, 16, 11, 0),
    (100, 50, 40, 2, 0),     # zeta > 32: generic sequential path
    (4000, 128, 8, 3, 123456789),  # a window of global columns
    (70000, 64, 12, 99, 5),  # d > 65535 (wide row ids)
]

STATS_CASES = [  # RejectionStats only (Appendix A)
    (4000, 1000000, 8, 11),
    (2000, 1000000, 16, 11),
    (400, 20000, 8, 3),
]


def main() -> None:
    os.makedirs(OUT, exist_ok=True)
    R = oracle.REF()
    meta = {"generator": "tools/make_golden.py", "source": "oracle/_ref (reference headers compiled in place)"}

    # rng.hpp KATs
    rng = {
        "seed0": R.rng_draws(0, None, 8),
        "s42_0": R.rng_draws(42, 0, 8),
        "s42_1": R.rng_draws(42, 1, 8),
        "ub_7_10_16": R.uniform_below(7, 10, 16, 64),
        "ub_3_4_4000": R.uniform_below(3, 4, 4000, 64),
    }
    np.savez_compressed(os.path.join(OUT, "rng.npz"), **rng)

    arrays = {}
    cases = []
    for i, (d, m, z, s, cb) in enumerate(SKETCH_CASES):
        rows, vals, colptr, st = R.generate_sparse_sign(d, m, z, s, col_begin=cb)
        arrays[f"rows_{i}"] = rows
        arrays[f"vals_{i}"] = vals
        arrays[f"colptr_{i}"] = colptr
        cases.append({"d": d, "m": m, "zeta": z, "seed": s, "col_begin": cb,
                      "columns_resampled": st[0], "resample_rounds": st[1]})
    np.savez_compressed(os.path.join(OUT, "sketch.npz"), **arrays)

    stats = []
    for d, m, z, s in STATS_CASES:
        _, _, _, st = R.generate_sparse_sign(d, m, z, s)
        stats.append({"d": d, "m": m, "zeta": z, "seed": s, "columns_resampled": st[0],
                      "resample_rounds": st[1]})

    # One small solve pipeline, every intermediate (sketch.hpp:297/304,
    # qr.hpp:21, triangular.hpp:14, preconditioner.hpp:48, lsqr.hpp:175/185).
    m, n, d, z = 600, 24, 96, 6
    A = R.gen_dense(m, n, 1e3, 91)
    b, xs = R.gen_rhs(A, 0.5, 92)
    Y, Sb = R.sketch_apply(d, z, 93, A, b)
    Q, Rf = R.householder_qr(Y)
    M = R.tri_inverse(Rf)
    M2, Q2, x0, _ = R.build_preconditioner(Y, Sb)
    assert np.array_equal(M, M2) and np.array_equal(Q, Q2)
    x_std, rep_std = R.lsqr(A, M, b, x0, eps=0.0, maxit=12, one_sync=False, x_star=xs, track_true=True)
    x_one, rep_one = R.lsqr(A, M, b, x0, eps=0.0, maxit=12, one_sync=True, x_star=xs, track_true=True)
    x_tol, rep_tol = R.lsqr(A, M, b, np.zeros(n), eps=1e-10, maxit=100, one_sync=False)
    np.savez_compressed(
        os.path.join(OUT, "pipeline.npz"), A=A, b=b, x_star=xs, Y=Y, Sb=Sb, Q=Q, R=Rf, M=M, x0=x0,
        x_std=x_std, est_std=rep_std.residual_estimate, err_std=rep_std.iterates_error,
        true_std=rep_std.residual_true, x_one=x_one, est_one=rep_one.residual_estimate,
        x_tol=x_tol, est_tol=rep_tol.residual_estimate,
    )
    pipeline = {"m": m, "n": n, "d": d, "zeta": z, "cond": 1e3, "seed_A": 91, "seed_b": 92,
                "seed_S": 93, "rho": 0.5, "maxit": 12,
                "tol_run": {"iterations": rep_tol.iterations, "termination": rep_tol.termination}}

    # Gradient family on the same problem (gradient.hpp:27-126): heavy ball
    # with hbm_params(eta) and plain descent with gd_params(eta), eta = sqrt(n/d)
    eta = float(np.sqrt(n / d))
    a_h, b_h = R.gradient_params(eta, True)
    a_g, b_g = R.gradient_params(eta, False)
    x_hbm, rep_hbm = R.gd_hbm(A, M, b, x0, a_h, b_h, eps=0.0, maxit=15, x_star=xs, track_true=True)
    x_gd, rep_gd = R.gd_hbm(A, M, b, x0, a_g, b_g, eps=0.0, maxit=15)
    x_ht, rep_ht = R.gd_hbm(A, M, b, x0, a_h, b_h, eps=1e-8, maxit=200)
    np.savez_compressed(
        os.path.join(OUT, "gradient.npz"), x_hbm=x_hbm, est_hbm=rep_hbm.residual_estimate,
        err_hbm=rep_hbm.iterates_error, true_hbm=rep_hbm.residual_true, x_gd=x_gd, est_gd=rep_gd.residual_estimate,
        x_ht=x_ht, est_ht=rep_ht.residual_estimate,
    )
    gradient = {"eta": eta, "hbm": [a_h, b_h], "gd": [a_g, b_g], "maxit": 15,
                "tol_run": {"eps": 1e-8, "iterations": rep_ht.iterations, "termination": rep_ht.termination}}

    # Distributed (distsim.hpp) partition + bit-identity across p
    parts = {str(p): R.partition_rows(333, p).tolist() for p in (1, 2, 4, 8)}
    parts.update({"4000000/8": R.partition_rows(4_000_000, 8).tolist(),
                  "1048576/3": R.partition_rows(1 << 20, 3).tolist()})

    meta.update({"sketch_cases": cases, "stats_cases": stats, "pipeline": pipeline,
                 "gradient": gradient, "partition_rows": parts})
    with open(os.path.join(OUT, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
