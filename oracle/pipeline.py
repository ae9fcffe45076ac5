"""ORACLE (test infrastructure only) — the confidence-region pipeline of Alg. 1,
step by step in the paper's order, calling the plain C loops in oracle/csrc/oracle.c.

Steps (readings R1-R18 in DESIGN.md):
  O1 marginal_order : p_M = 1 - Phi((u - mu)/sqrt(Sigma_ii)) (Alg. 1 l.3-5), descending
                      order (l.6); sort key z = (mu - u)/sqrt(Sigma_ii), ties by ascending index
                      (R13); limits a_k = u - mu_o(k), b_k = +inf (R2).
  O2 covariance     : oracle/matern.py (Eq. 6).
  O3 cholesky       : textbook Crout (C).
  O4 lattice        : oracle/lattice.py (R8).
  O5 sov_units      : per-sample SOV sweep (C), one log weight per (prefix, sample) (R1, R9, R10).
  O6 prefix_logp    : log P_k = M_k + log sum exp(ell - M_k) - log(N R)  (mean(p), Alg. 2 l.19; R11).
  O7 region         : running min, k*(c) = max{k : log P_k >= log c} (Eq. 4-5; R12, R16).
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import lib, ptr
from .lattice import generators, shifts
from .matern import covariance


def Phi(x: float) -> float:
    return lib().orc_Phi(float(x))


def Phibar(x: float) -> float:
    return lib().orc_Phibar(float(x))


def Phiinv(p: float) -> float:
    """Phi^{-1}(p) on (0,1) via the lower-half Halley solver and symmetry."""
    p = float(p)
    return lib().orc_Phiinv_lower(p) if p <= 0.5 else -lib().orc_Phiinv_lower(1.0 - p)


def sov_step(ap: float, bp: float, w: float) -> tuple[float, float]:
    lq = ctypes.c_double()
    y = ctypes.c_double()
    lib().orc_sov_step(float(ap), float(bp), float(w), ctypes.byref(lq), ctypes.byref(y))
    return lq.value, y.value


def cholesky(S: np.ndarray, nthreads: int = 0) -> tuple[np.ndarray, int]:
    """Returns (L, info): L lower (upper triangle zeroed), info = -1 ok else 0-based failing row."""
    A = np.array(S, dtype=np.float64, order="C", copy=True)
    n = A.shape[0]
    info = lib().orc_cholesky(n, ptr(A), int(nthreads))
    return np.tril(A), int(info)


def marginal_order(mu: np.ndarray, var_diag: np.ndarray, u: float):
    """O1. Returns (order, a_sorted, pM) — order[k] is the original index of sorted position k."""
    mu = np.asarray(mu, dtype=np.float64)
    z = (mu - u) / np.sqrt(np.asarray(var_diag, dtype=np.float64))
    order = np.argsort(-z, kind="stable")
    a = u - mu[order]
    pM = np.array([Phi(v) for v in z])
    return order.astype(np.int64), a, pM


def sov_unit(L: np.ndarray, a, b, G, D_r, j0: int, J: int, want_ell=False, want_y=False):
    """One unit (shift with shifts D_r, lattice indices j0..j0+J-1). Returns (MS[n,2], ell[n,J]?, y[n,J]?)."""
    L = np.ascontiguousarray(L, dtype=np.float64)
    n = L.shape[0]
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    G = np.ascontiguousarray(G, dtype=np.uint64)
    D_r = np.ascontiguousarray(D_r, dtype=np.uint64)
    MS = np.empty((n, 2))
    ell = np.empty((n, J)) if want_ell else None
    y = np.empty((n, J)) if want_y else None
    rc = lib().orc_sov_unit(n, ptr(L), n, ptr(a), ptr(b), ptr(G), ptr(D_r), int(j0), int(J), ptr(MS),
                            ptr(ell) if ell is not None else None, ptr(y) if y is not None else None)
    assert rc == 0
    return MS, ell, y


def sov_units(L: np.ndarray, a, b, G, D, N: int, R: int, chunk: int, unit_begin: int = 0,
              unit_end: int | None = None, nthreads: int = 0) -> np.ndarray:
    """O5 over units u in [unit_begin, unit_end), ordered (r, c). Returns partials [units][n][2]."""
    L = np.ascontiguousarray(L, dtype=np.float64)
    n = L.shape[0]
    C = -(-N // chunk)
    if unit_end is None:
        unit_end = R * C
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    G = np.ascontiguousarray(G, dtype=np.uint64)
    D = np.ascontiguousarray(D, dtype=np.uint64)
    out = np.empty((unit_end - unit_begin, n, 2))
    rc = lib().orc_sov_units(n, ptr(L), n, ptr(a), ptr(b), ptr(G), ptr(D), int(N), int(R), int(chunk),
                             int(unit_begin), int(unit_end), ptr(out), int(nthreads))
    assert rc == 0
    return out


def combine_units(partials: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """(M_k, S_k) over units in ascending unit order: M = max_u M_u, S = sum_u S_u exp(M_u - M)."""
    P = np.asarray(partials)
    M = np.max(P[:, :, 0], axis=0)
    S = np.zeros(P.shape[1])
    for u in range(P.shape[0]):
        Mu, Su = P[u, :, 0], P[u, :, 1]
        with np.errstate(invalid="ignore"):
            t = np.where(Mu == -np.inf, 0.0, Su * np.exp(Mu - M))
        S = S + t
    return M, S


def prefix_logp(M: np.ndarray, S: np.ndarray, NR: int) -> np.ndarray:
    """O6: log P_k = M_k + log S_k - log(NR) (mean over all N*R samples, R11)."""
    with np.errstate(divide="ignore"):
        return np.where(S > 0, M + np.log(S) - math.log(NR), -np.inf)


def per_shift_logp(partials: np.ndarray, N: int, R: int, chunk: int) -> np.ndarray:
    """log P^(r)_k per shift r (for the standard error across shifts, R11). Needs all units."""
    C = -(-N // chunk)
    out = []
    for r in range(R):
        M, S = combine_units(partials[r * C:(r + 1) * C])
        out.append(prefix_logp(M, S, N))
    return np.array(out)


def shift_stats(logp_shift: np.ndarray):
    """O6: from the per-shift estimates log P^(r)_k (R x n, equal N per shift) the
    combined log P_k = log(mean_r P^(r)_k) (= the mean over all N R samples, R11) and the relative
    standard error across the R randomised shifts, sd_r(P^(r)_k) / (sqrt(R) mean_r P^(r)_k) (ddof 1)
    — the QMC error estimate of randomly shifted lattice rules; about the standard error of log P_k.
    Evaluated relative to max_r log P^(r)_k, so P far below the double range is no problem."""
    L = np.asarray(logp_shift, dtype=np.float64)
    R = L.shape[0]
    m = np.max(L, axis=0)
    with np.errstate(invalid="ignore", divide="ignore"):
        x = np.where(np.isfinite(m), np.exp(L - m), 0.0)          # P^(r) / max_r P^(r)
        xm = np.mean(x, axis=0)
        logp = np.where(xm > 0, m + np.log(xm), -np.inf)
        sd = np.std(x, axis=0, ddof=1) if R > 1 else np.zeros_like(xm)
        rel = np.where(xm > 0, sd / (math.sqrt(R) * xm), np.nan)
    return logp, rel


def region(logp: np.ndarray, conf, tie_tol: float = 1e-8):
    """O7: running min (R12), k*(c) = max{k : log P_k >= log c} (Eq. 4), near-tie flags."""
    lp = np.minimum.accumulate(np.asarray(logp, dtype=np.float64))
    ks, ties = [], []
    for c in conf:
        lc = math.log(c)
        k = int(np.count_nonzero(lp >= lc))
        tie = (k > 0 and abs(lp[k - 1] - lc) <= tie_tol) or (k < len(lp) and abs(lp[k] - lc) <= tie_tol)
        ks.append(k)
        ties.append(bool(tie))
    return np.array(ks, dtype=np.int64), np.array(ties)


@dataclass
class CrdResult:
    order: np.ndarray
    a: np.ndarray
    L: np.ndarray
    logp: np.ndarray
    k_star: np.ndarray
    near_tie: np.ndarray
    partials: np.ndarray
    info: int


def crd(xy, mu, sigma2, beta, nu, nugget, u, N, R, seed, conf, chunk=None, nthreads=0, L=None):
    """Alg. 1 end to end (small n). If L (sorted order) is given, steps O2-O3 are skipped (shared-L mode)."""
    xy = np.asarray(xy, dtype=np.float64)
    n = xy.shape[0]
    var = np.full(n, sigma2 + nugget)
    order, a, _ = marginal_order(mu, var, u)
    info = -1
    if L is None:
        S = covariance(xy[order], sigma2, beta, nu, nugget)
        L, info = cholesky(S, nthreads)
        if info >= 0:
            raise FloatingPointError(f"Sigma not positive definite at row {info}")
    b = np.full(n, np.inf)
    G = generators(n)
    D = shifts(seed, R, n)
    chunk = chunk or N
    parts = sov_units(L, a, b, G, D, N, R, chunk, nthreads=nthreads)
    M, Ssum = combine_units(parts)
    logp = prefix_logp(M, Ssum, N * R)
    ks, ties = region(logp, conf)
    return CrdResult(order, a, L, logp, ks, ties, parts, info)


def crd_cov(Sigma, mu, u, N, R, seed, conf, chunk=None, nthreads=0):
    """Alg. 1 end to end for a given covariance in the original site order (e.g. Sigma_post of
    Eq. 7 with mu_post of Eq. 8): marginals from diag(Sigma), order, Sigma permuted to sorted
    order (R1), Cholesky, one sweep, regions."""
    Sigma = np.asarray(Sigma, dtype=np.float64)
    n = Sigma.shape[0]
    order, a, _ = marginal_order(mu, np.diag(Sigma).copy(), u)
    L, info = cholesky(Sigma[np.ix_(order, order)], nthreads)
    if info >= 0:
        raise FloatingPointError(f"Sigma not positive definite at row {info}")
    b = np.full(n, np.inf)
    G = generators(n)
    D = shifts(seed, R, n)
    chunk = chunk or N
    parts = sov_units(L, a, b, G, D, N, R, chunk, nthreads=nthreads)
    M, Ssum = combine_units(parts)
    logp = prefix_logp(M, Ssum, N * R)
    ks, ties = region(logp, conf)
    return CrdResult(order, a, L, logp, ks, ties, parts, info)
