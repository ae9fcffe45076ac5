"""ORACLE (test infrastructure only) — Matérn covariance, Eq. 6, written out literally:

    C(h; sigma^2, a, nu) = sigma^2 / (2^(nu-1) Gamma(nu)) * (h/a)^nu * K_nu(h/a),   C(0) = sigma^2

with K_nu the modified Bessel function of the second kind (scipy.special.kv, a library primitive
used as one step) — note: no sqrt(2 nu) scaling, exactly as the paper prints it (reading R14).
Euclidean distance; nugget added to the diagonal only (R14).
"""
from __future__ import annotations

import numpy as np
from scipy.special import gamma, kv


def matern(h, sigma2: float, beta: float, nu: float) -> np.ndarray:
    h = np.asarray(h, dtype=np.float64)
    x = h / beta
    out = np.empty_like(x)
    pos = x > 0
    xp = x[pos]
    out[pos] = sigma2 / (2.0 ** (nu - 1.0) * gamma(nu)) * xp ** nu * kv(nu, xp)
    out[~pos] = sigma2
    return out


def covariance(xy: np.ndarray, sigma2: float, beta: float, nu: float, nugget: float) -> np.ndarray:
    """Dense Sigma (Alg. 1 line 2) for the given (already sorted) locations, row-major n x n.

    Sigma_kl = C(||x_k - x_l||_2) + nugget * delta_kl, computed once per unordered pair so that it is
    exactly symmetric.
    """
    xy = np.asarray(xy, dtype=np.float64)
    n = xy.shape[0]
    S = np.empty((n, n), dtype=np.float64)
    for k in range(n):
        dx = xy[k, 0] - xy[: k + 1, 0]
        dy = xy[k, 1] - xy[: k + 1, 1]
        h = np.sqrt(dx * dx + dy * dy)
        row = matern(h, sigma2, beta, nu)
        S[k, : k + 1] = row
        S[: k + 1, k] = row
    S[np.arange(n), np.arange(n)] += nugget
    return S
