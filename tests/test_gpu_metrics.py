"""GPU checks of the sketch-quality metrics (metrics.hpp):
S U and the QR factorizations run on the B200; the reference's distortion
(compiled, oracle/_ref) is the bar when present, numpy otherwise."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

slq = pytest.importorskip("paper_2506_03070_b200")
A = slq.analysis


def _basis(m, n, seed):
    rng = np.random.default_rng(seed)
    return np.linalg.qr(rng.standard_normal((m, n)))[0]


@pytest.mark.parametrize("m,n,d,zeta", [(2000, 20, 80, 8), (5000, 40, 400, 4), (1000, 10, 30, 2)])
def test_distortion_vs_reference(m, n, d, zeta):
    U = _basis(m, n, m)
    S = slq.generate_sparse_sign(d, m, zeta, 11)
    rep = A.distortion(S, U)
    sv = np.linalg.svd(S.matrix.todense() @ U, compute_uv=False)
    assert abs(rep.sigma_max - sv[0]) <= 1e-12 and abs(rep.sigma_min - sv[-1]) <= 1e-12
    assert rep.eta == max(1 - rep.sigma_min, rep.sigma_max - 1) and rep.d == d and rep.zeta == zeta
    b = np.random.default_rng(1).standard_normal(m)
    rep_b = A.distortion(S, U, also_b=b)
    assert rep_b.eta >= rep.eta - 1e-12  # a larger subspace cannot distort less
    if oracle.ref_available():
        R = oracle.REF()
        for got, bb in ((rep, None), (rep_b, b)):
            eta, smin, smax = R.distortion(d, zeta, 11, U, bb)
            # the reference takes sqrt of Gram eigenvalues (Jacobi): ~1e-14 relative at sigma ~ 1
            assert abs(got.eta - eta) <= 1e-10 and abs(got.sigma_min - smin) <= 1e-10 and abs(got.sigma_max - smax) <= 1e-10


def test_trials_spectrum_coherence():
    m, n, d = 4000, 20, 160
    U = _basis(m, n, 3)

    def apply_sketch(Ub, t):
        return slq.apply(slq.generate_sparse_sign(d, m, 8, 100 + t), Ub)

    rep = A.distortion_trials(apply_sketch, U, 9)
    singles = [A.distortion(slq.generate_sparse_sign(d, m, 8, 100 + t), U).eta for t in range(9)]
    assert rep.trials == 9 and rep.q50 == rep.eta == A.quantile(singles, 0.5)
    assert rep.q05 <= rep.q50 <= rep.q95
    assert 0.2 < rep.eta < 0.8  # ~ sqrt(n/d) = 0.35 for a sparse sign sketch
    h = A.sketched_spectrum(apply_sketch, U, 4, bins=30)
    assert sum(h.counts) == 4 * n and len(h.bin_edges) == 31 and len(h.overlay) == 30
    assert max(h.overlay) > 0
    # leverage scores of a coherent matrix: identity rows on top of noise
    B = np.vstack([np.eye(n), 1e-3 * np.random.default_rng(4).standard_normal((m - n, n))])
    cs = A.coherence_stats(B)
    assert abs(cs.sum - n) <= 1e-9 and cs.max > 0.99 and cs.median < 1e-3
    Q = A.orthonormal_basis(B)
    assert np.abs(Q.T @ Q - np.eye(n)).max() <= 1e-12
