"""ORACLE (test infrastructure only) — NEXT-4, posterior conditioning of the field before Alg. 1.

PAPER.md §V-A: m noisy observations y = A x + N(0, tau^2 I) (A the m x n indicator
matrix of the observed sites, tau = 0.5 in the paper) give
    Sigma_post = (Sigma^{-1} + (1/tau^2) A^T A)^{-1}                      (Eq. 7)
    mu_post    = mu + (1/tau^2) Sigma_post A^T (y - A mu)                 (Eq. 8)
and "Sigma_post can be used as input to Algorithm 1 (line 2) and mu_post ... to update the a
vector". Written out literally with dense inverses (numpy.linalg.inv), in fp64, for the
small n the tests use. Pinned in tests/test_oracle_posterior.py against the scalar conjugate-normal
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
    """Eq. 7 and Eq. 8 literally. Returns (Sigma_post, mu_post)."""
    n = Sigma.shape[0]
    A = indicator(obs, n)
    P = np.linalg.inv(Sigma) + (1.0 / tau ** 2) * (A.T @ A)
    Sp = np.linalg.inv(P)
    Sp = 0.5 * (Sp + Sp.T)
    mp = mu + (1.0 / tau ** 2) * (Sp @ (A.T @ (y - A @ mu)))
    return Sp, mp


def posterior_field(xy: np.ndarray, mu: np.ndarray, obs: np.ndarray, y: np.ndarray, sigma2: float, beta: float,
                    nu: float, nugget: float, tau: float):
    """Eq. 6 covariance of the sites, then Eq. 7-8."""
    S = covariance(xy, sigma2, beta, nu, nugget)
    return posterior(S, mu, obs, y, tau)
