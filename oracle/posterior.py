"""ORACLE (test infrastructure only) — NEXT-4, posterior conditioning of the field before Alg. 1.

PAPER.md §V-A: m noisy observations y = A x + N(0, tau^2 I) (A the m x n indicator
matrix of the observed sites, tau = 0.5 in the paper) give
    Sigma_post = (Sigma^{-1} + (1/tau^2) A^T A)^{-1}                      (Eq. 7)
    mu_post    = mu + (1/tau^2) Sigma_post A^T (y - A mu)                 (Eq. 8)
and "Sigma_post can be used as input to Algorithm 1 (line 2) and mu_post ... to update the a
vector". Eq. 7 is evaluated as (I + Sigma B)^{-1} Sigma with B = tau^{-2} A^T A — the
push-through form of the same inverse, (Sigma^{-1} + B)^{-1} = (I + Sigma B)^{-1} Sigma, which
avoids inverting Sigma itself (cond(Sigma) reaches 1e7 for nu = 3/2; cond(I + Sigma B) <=
1 + lambda_max(Sigma_oo)/tau^2) — with one dense LU solve (numpy.linalg.solve), fp64, for the small
n the tests use. Eq. 8 is then applied as printed. Pinned in tests/test_oracle_posterior.py against the scalar conjugate-normal
closed form, the conditional-Gaussian (Woodbury) form, and limiting cases.
"""
from __future__ import annotations

import numpy as np

from .matern import covariance


def indicator(obs: np.ndarray, n: int) -> np.ndarray:
    """A (m x n): A[r, obs[r]] = 1."""
    A = np.zeros((len(obs), n))
    A[np.arange(len(obs)), obs] = 1.0
    return A


def posterior(Sigma: np.ndarray, mu: np.ndarray, obs: np.ndarray, y: np.ndarray, tau: float):
    """Eq. 7 (push-through form, see the module docstring) and Eq. 8. Returns (Sigma_post, mu_post)."""
    n = Sigma.shape[0]
    A = indicator(obs, n)
    B = (1.0 / tau ** 2) * (A.T @ A)
    Sp = np.linalg.solve(np.eye(n) + Sigma @ B, Sigma)
    Sp = 0.5 * (Sp + Sp.T)
    mp = mu + (1.0 / tau ** 2) * (Sp @ (A.T @ (y - A @ mu)))
    return Sp, mp


def posterior_literal(Sigma: np.ndarray, mu: np.ndarray, obs: np.ndarray, y: np.ndarray, tau: float):
    """Eq. 7 with explicit inverses exactly as printed (pin only: accurate to ~cond(Sigma)^2 eps)."""
    n = Sigma.shape[0]
    A = indicator(obs, n)
    Sp = np.linalg.inv(np.linalg.inv(Sigma) + (1.0 / tau ** 2) * (A.T @ A))
    mp = mu + (1.0 / tau ** 2) * (Sp @ (A.T @ (y - A @ mu)))
    return Sp, mp


def posterior_field(xy: np.ndarray, mu: np.ndarray, obs: np.ndarray, y: np.ndarray, sigma2: float, beta: float,
                    nu: float, nugget: float, tau: float):
    """Eq. 6 covariance of the sites, then Eq. 7-8."""
    S = covariance(xy, sigma2, beta, nu, nugget)
    return posterior(S, mu, obs, y, tau)
