"""Host-side companions of the solver path:

* embedding-dimension planner  -- embedding.hpp:13-100
* sketch-quality metrics       -- metrics.hpp:17-231 (the sketch products S U
  and the QR factorizations run on the B200 through the library; only n x n
  singular values and scalar statistics are computed on the host)
* Matrix Market exchange       -- matrix_market.hpp:17-170

Names, argument meaning and error types follow the reference.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from .api import (
    CscMatrix,
    DimensionMismatch,
    Error,
    InvalidDims,
    InvalidDistortion,
    SparseSignSketch,
    apply,
    householder_qr,
)


class NegativeArgument(Error):
    """errors.hpp:49"""


class InvalidResidual(Error):
    """errors.hpp:54"""


class UnsupportedFormat(Error):
    """errors.hpp:59"""


# ------------------------------------------------------------ embedding.hpp


@dataclass
class RateEstimate:
    """embedding.hpp:13-16"""

    rate_per_iter: float
    kappa: float


def estimate_rate(n: int, d: int) -> RateEstimate:
    """embedding.hpp:20-24: rate sqrt(n/d), kappa = (1+r)/(1-r)."""
    if d <= n:
        raise InvalidDims("estimate_rate: need d > n")
    r = math.sqrt(n / d)
    return RateEstimate(r, (1.0 + r) / (1.0 - r))


def iterations_for(eps: float, n: int, d: int) -> int:
    """embedding.hpp:28-35: ceil(log eps / log(n/d)), at least 1."""
    if d <= n:
        raise InvalidDims("iterations_for: need d > n")
    if eps >= 1.0:
        return 1
    ratio = math.log(eps) / math.log(n / d)
    return max(1, int(math.ceil(ratio - 1e-9)))


def lambert_w(x: float) -> float:
    """embedding.hpp:40-61: principal branch, safeguarded Halley iteration."""
    if x < 0.0:
        raise NegativeArgument("lambert_w: argument must be >= 0")
    if x == 0.0:
        return 0.0
    lo, hi = 0.0, math.log1p(x) + 1.0
    w = math.log1p(x)
    for _ in range(200):
        ew = math.exp(w)
        f = w * ew - x
        if abs(f) <= 1e-13 * max(1.0, x):
            break
        if f > 0.0:
            hi = w
        else:
            lo = w
        fp = ew * (w + 1.0)
        fpp = ew * (w + 2.0)
        nxt = w - f / (fp - 0.5 * f * fpp / fp)
        if not (lo < nxt < hi):
            nxt = 0.5 * (lo + hi)
        w = nxt
    return w


@dataclass
class DimensionPlan:
    """embedding.hpp:64-69"""

    d: int = 0
    predicted_iters: int = 0
    predicted_kappa: float = 0.0
    eps: float = 0.0


def balance_dimension_real(m: int, n: int, eps: float) -> float:
    """embedding.hpp:74-80: d = n exp(W(-m log(eps) / n^2))."""
    if not (m > n >= 1):
        raise InvalidDims("balance_dimension_real: need m > n >= 1")
    if not (0.0 < eps < 1.0):
        raise InvalidDims("balance_dimension_real: need 0 < eps < 1")
    return n * math.exp(lambert_w(-m * math.log(eps) / (float(n) * float(n))))


def select_embedding_dim(m: int, n: int, eps: float) -> DimensionPlan:
    """embedding.hpp:84-98: balance point rounded half up, clamped to [n+1, m]."""
    d = int(math.floor(balance_dimension_real(m, n, eps) + 0.5))
    d = min(max(d, n + 1), m)
    return DimensionPlan(d, iterations_for(eps, n, d), estimate_rate(n, d).kappa, eps)


# -------------------------------------------------------------- metrics.hpp


@dataclass
class DistortionReport:
    """metrics.hpp:18-26"""

    eta: float = 0.0
    sigma_min: float = 0.0
    sigma_max: float = 0.0
    d: int = 0
    zeta: int = 0
    trials: int = 1
    q05: float = 0.0
    q50: float = 0.0
    q95: float = 0.0


def singular_values(B, ctx=None) -> np.ndarray:
    """Descending singular values of a tall B (eigen_sym.hpp:69-82 computes them
    from the Gram matrix; here from the device QR's R, which loses nothing for
    small singular values)."""
    B = np.asarray(B, dtype=np.float64)
    if B.shape[0] < B.shape[1]:
        raise DimensionMismatch("singular_values: need rows >= cols")
    R = householder_qr(B, ctx=ctx).R
    return np.linalg.svd(R, compute_uv=False)


def orthonormal_basis(A, ctx=None) -> np.ndarray:
    """metrics.hpp:29-30: Q of the thin Householder QR (device)."""
    if isinstance(A, CscMatrix):
        A = A.todense()
    return householder_qr(A, ctx=ctx).Q


def extend_basis(U, b) -> np.ndarray:
    """metrics.hpp:50-61: append the normalized component of b outside range(U)."""
    U = np.asarray(U, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    res = b - U @ (U.T @ b)
    rn = np.linalg.norm(res)
    if rn <= 1e-12 * np.linalg.norm(b):
        return U
    return np.column_stack([U, res / rn])


def _single(SU, ctx=None):
    sv = singular_values(SU, ctx=ctx)
    smax, smin = float(sv[0]), float(sv[-1])
    return max(1.0 - smin, smax - 1.0), smin, smax


def distortion(S: SparseSignSketch, U, also_b=None, ctx=None) -> DistortionReport:
    """metrics.hpp:66-78: distortion of one sketch on range(U) (+ span(b)).
    S U is formed on the B200 (bit-identical to the reference's apply)."""
    basis = extend_basis(U, also_b) if also_b is not None else np.asarray(U, dtype=np.float64)
    eta, smin, smax = _single(apply(S, basis, ctx=ctx), ctx)
    return DistortionReport(eta, smin, smax, d=S.matrix.rows, zeta=S.zeta, trials=1, q05=eta, q50=eta, q95=eta)


def quantile(v, q: float) -> float:
    """metrics.hpp:84-92: linear interpolation between order statistics."""
    v = sorted(v)
    if not v:
        return 0.0
    pos = q * (len(v) - 1.0)
    lo = int(pos)
    hi = min(lo + 1, len(v) - 1)
    frac = pos - lo
    return v[lo] * (1.0 - frac) + v[hi] * frac


def distortion_trials(apply_sketch: Callable[[np.ndarray, int], np.ndarray], U, trials: int,
                      ctx=None) -> DistortionReport:
    """metrics.hpp:95-118: median / 5% / 95% distortion over independent draws;
    apply_sketch(U, trial) returns S_trial U."""
    singles = [_single(apply_sketch(U, t), ctx) for t in range(trials)]
    etas = [s[0] for s in singles]
    med = quantile(etas, 0.5)
    best = 0
    for i in range(1, len(singles)):
        if abs(singles[i][0] - med) < abs(singles[best][0] - med):
            best = i
    return DistortionReport(med, singles[best][1], singles[best][2], trials=trials, q05=quantile(etas, 0.05),
                            q50=med, q95=quantile(etas, 0.95))


def marchenko_pastur_pdf(x: float, ratio: float) -> float:
    """metrics.hpp:122-130"""
    if not (0.0 < ratio <= 1.0):
        raise InvalidDims("marchenko_pastur_pdf: ratio in (0,1]")
    if not x > 0.0:
        return 0.0
    sr = math.sqrt(ratio)
    lm, lp = (1.0 - sr) ** 2, (1.0 + sr) ** 2
    if x <= lm or x >= lp:
        return 0.0
    return math.sqrt((lp - x) * (x - lm)) / (2.0 * math.pi * ratio * x)


def cond_bound(eta: float) -> float:
    """metrics.hpp:133-136: cond(AM) <= (1 + eta) / (1 - eta)."""
    if not (0.0 <= eta < 1.0):
        raise InvalidDistortion("cond_bound: need 0 <= eta < 1")
    return (1.0 + eta) / (1.0 - eta)


def forward_error_from_residuals(res_hat: float, res_star: float) -> float:
    """metrics.hpp:141-150"""
    if res_star < 0.0 or res_hat < 0.0:
        raise InvalidResidual("forward_error_from_residuals: negative residual norm")
    if res_hat < res_star * (1.0 - 1e-12) - 1e-12:
        raise InvalidResidual("forward_error_from_residuals: res_hat < res_star")
    diff = res_hat * res_hat - res_star * res_star
    return math.sqrt(diff) if diff > 0.0 else 0.0


@dataclass
class CoherenceStats:
    """metrics.hpp:153-156"""

    min: float = 0.0
    q25: float = 0.0
    median: float = 0.0
    q75: float = 0.0
    max: float = 0.0
    sum: float = 0.0


def coherence_stats(A, ctx=None) -> CoherenceStats:
    """metrics.hpp:158-176: leverage scores ||U[i,:]||^2 of the device QR basis."""
    U = orthonormal_basis(A, ctx=ctx)
    scores = np.einsum("ij,ij->i", U, U)
    s = list(scores)
    return CoherenceStats(float(scores.min()), quantile(s, 0.25), quantile(s, 0.5), quantile(s, 0.75),
                          float(scores.max()), float(scores.sum()))


@dataclass
class SpectrumHistogram:
    """metrics.hpp:181-185"""

    bin_edges: list = field(default_factory=list)
    counts: list = field(default_factory=list)
    overlay: list = field(default_factory=list)


def sketched_spectrum(apply_sketch: Callable[[np.ndarray, int], np.ndarray], U, trials: int, bins: int = 50,
                      ctx=None) -> SpectrumHistogram:
    """metrics.hpp:187-221: histogram of sigma_i(S U)^2 over trials with the
    Marchenko-Pastur density at the bin centres."""
    U = np.asarray(U, dtype=np.float64)
    vals = []
    d = 0
    for t in range(trials):
        SU = apply_sketch(U, t)
        d = SU.shape[0]
        vals.extend(float(s) * float(s) for s in singular_values(SU, ctx=ctx))
    ratio = U.shape[1] / d
    sr = math.sqrt(ratio)
    lo = max(0.0, (1.0 - sr) ** 2 - 0.25 * sr)
    hi_edge = (1.0 + sr) ** 2 + 0.25 * sr
    lo_edge = min(lo, min(vals))
    hi = max(hi_edge, max(vals) + 1e-12)
    h = SpectrumHistogram()
    h.bin_edges = [lo_edge + (hi - lo_edge) * i / bins for i in range(bins + 1)]
    h.counts = [0] * bins
    for v in vals:
        idx = int((v - lo_edge) / (hi - lo_edge) * bins)
        h.counts[min(max(idx, 0), bins - 1)] += 1
    for i in range(bins):
        c = 0.5 * (h.bin_edges[i] + h.bin_edges[i + 1])
        h.overlay.append(marchenko_pastur_pdf(c, ratio) if c > 0.0 else 0.0)
    return h


# ------------------------------------------------------- matrix_market.hpp


def _read_header(f, path):
    line = f.readline()
    if not line:
        raise UnsupportedFormat(f"{path}: empty file")
    parts = (line.split() + [""] * 5)[:5]
    banner, obj, fmt, fld, sym = (p.lower() for p in parts)
    if banner != "%%matrixmarket" or obj != "matrix":
        raise UnsupportedFormat(f"{path}: missing MatrixMarket matrix banner")
    if fmt not in ("coordinate", "array"):
        raise UnsupportedFormat(f"{path}: format '{fmt}' not supported")
    if fld != "real":
        raise UnsupportedFormat(f"{path}: field '{fld}' not supported (real only)")
    if sym != "general":
        raise UnsupportedFormat(f"{path}: symmetry '{sym}' not supported")
    return fmt == "coordinate"


def _size_line(f):
    for line in f:
        if line.strip() and not line.startswith("%"):
            return line.split()
    return []


def _tokens(f):
    for line in f:
        yield from line.split()


def read_csc(path: str) -> CscMatrix:
    """matrix_market.hpp:64-107: coordinate file -> CSC (1-based on disk,
    duplicates summed, rows sorted within each column)."""
    try:
        f = open(path)
    except OSError:
        raise Error(f"cannot open {path}") from None
    with f:
        if not _read_header(f, path):
            raise UnsupportedFormat(f"{path}: expected coordinate format")
        sz = _size_line(f)
        try:
            rows, cols, nnz = int(sz[0]), int(sz[1]), int(sz[2])
        except (IndexError, ValueError):
            raise UnsupportedFormat(f"{path}: bad size line") from None
        if rows <= 0 or cols <= 0 or nnz < 0:
            raise UnsupportedFormat(f"{path}: bad size line")
        tok = _tokens(f)
        trip = []
        try:
            for _ in range(nnz):
                i, j, v = int(next(tok)), int(next(tok)), float(next(tok))
                if not (1 <= i <= rows and 1 <= j <= cols):
                    raise UnsupportedFormat(f"{path}: entry index out of range")
                trip.append((j - 1, i - 1, v))
        except (StopIteration, ValueError):
            raise UnsupportedFormat(f"{path}: truncated entries") from None
    trip.sort(key=lambda t: (t[0], t[1]))
    ri, vals = [], []
    cp = np.zeros(cols + 1, np.int64)
    prev = (-1, -1)
    for j, i, v in trip:
        if (j, i) == prev:
            vals[-1] += v
            continue
        ri.append(i)
        vals.append(v)
        cp[j + 1] = len(vals)
        prev = (j, i)
    cp = np.maximum.accumulate(cp)
    return CscMatrix(rows, cols, np.array(vals, dtype=np.float64), np.array(ri, dtype=np.int64), cp)


def read_dense(path: str) -> np.ndarray:
    """matrix_market.hpp:110-128: array file -> dense column-major."""
    try:
        f = open(path)
    except OSError:
        raise Error(f"cannot open {path}") from None
    with f:
        if _read_header(f, path):
            raise UnsupportedFormat(f"{path}: expected array format")
        sz = _size_line(f)
        try:
            rows, cols = int(sz[0]), int(sz[1])
        except (IndexError, ValueError):
            raise UnsupportedFormat(f"{path}: bad size line") from None
        if rows <= 0 or cols <= 0:
            raise UnsupportedFormat(f"{path}: bad size line")
        tok = _tokens(f)
        out = np.empty(rows * cols)
        try:
            for k in range(rows * cols):
                out[k] = float(next(tok))
        except (StopIteration, ValueError):
            raise UnsupportedFormat(f"{path}: truncated entries") from None
    return out.reshape((rows, cols), order="F")


def load_matrix(path: str):
    """matrix_market.hpp:131-138: sniff the header, read either format."""
    try:
        f = open(path)
    except OSError:
        raise Error(f"cannot open {path}") from None
    with f:
        coord = _read_header(f, path)
    return read_csc(path) if coord else read_dense(path)


def _g17(v: float) -> str:
    return f"{v:.17g}"  # std::ostream precision(17), default float format


def write_csc(path: str, A: CscMatrix) -> None:
    """matrix_market.hpp:140-150"""
    try:
        f = open(path, "w")
    except OSError:
        raise Error(f"cannot open {path} for writing") from None
    with f:
        f.write("%%MatrixMarket matrix coordinate real general\n")
        f.write(f"{A.rows} {A.cols} {A.values.size}\n")
        cp = A.col_pointers
        for j in range(A.cols):
            for k in range(int(cp[j]), int(cp[j + 1])):
                f.write(f"{int(A.row_indices[k]) + 1} {j + 1} {_g17(float(A.values[k]))}\n")


def write_dense(path: str, A) -> None:
    """matrix_market.hpp:152-160"""
    A = np.asarray(A, dtype=np.float64)
    if A.ndim == 1:
        A = A.reshape(-1, 1)
    try:
        f = open(path, "w")
    except OSError:
        raise Error(f"cannot open {path} for writing") from None
    with f:
        f.write("%%MatrixMarket matrix array real general\n")
        f.write(f"{A.shape[0]} {A.shape[1]}\n")
        f.write("".join(_g17(float(v)) + "\n" for v in A.ravel(order="F")))


def write_vector(path: str, v) -> None:
    """matrix_market.hpp:162-166"""
    write_dense(path, np.asarray(v, dtype=np.float64).reshape(-1, 1))
