"""Pins of the oracle's NEXT-4 posterior conditioning (Eq. 7-8, oracle/posterior.py): the scalar
conjugate-normal closed form, the conditional-Gaussian (Woodbury) form of the same posterior,
unobserved blocks independent of the observations, and the noise-free / no-information limits.
CPU only."""
import numpy as np
import pytest

import oracle


def test_scalar_conjugate_normal():
    for s2, tau, mu, y in [(1.0, 0.5, 0.0, 1.2), (2.5, 1.5, -0.3, 0.4)]:
        Sp, mp = oracle.posterior(np.array([[s2]]), np.array([mu]), np.array([0]), np.array([y]), tau)
        assert Sp[0, 0] == pytest.approx(1.0 / (1.0 / s2 + 1.0 / tau ** 2), rel=1e-14)
        assert mp[0] == pytest.approx(mu + s2 / (s2 + tau ** 2) * (y - mu), rel=1e-13)


def test_matches_conditional_gaussian_form():
    """Sigma_post = Sigma - Sigma_{:,o} (Sigma_oo + tau^2 I)^{-1} Sigma_{o,:},
    mu_post = mu + Sigma_{:,o} (Sigma_oo + tau^2 I)^{-1} (y - mu_o)."""
    rng = np.random.default_rng(4)
    n, m, tau = 60, 17, 0.5
    xy = rng.uniform(size=(n, 2))
    S = oracle.covariance(xy, 1.0, 0.2, 1.5, 1e-8)
    mu = rng.standard_normal(n) * 0.3
    obs = np.sort(rng.choice(n, m, replace=False))
    y = rng.standard_normal(m)
    Sp, mp = oracle.posterior(S, mu, obs, y, tau)
    C = S[np.ix_(obs, obs)] + tau ** 2 * np.eye(m)
    K = S[obs, :]
    G = np.linalg.solve(C, K)
    assert np.max(np.abs(Sp - (S - K.T @ G))) <= 1e-12
    assert np.max(np.abs(mp - (mu + K.T @ np.linalg.solve(C, y - mu[obs])))) <= 1e-12


def test_matches_eq7_as_printed_on_a_well_conditioned_case():
    """The push-through evaluation equals Eq. 7 with explicit inverses where the latter is accurate."""
    rng = np.random.default_rng(8)
    n, m = 40, 9
    xy = rng.uniform(size=(n, 2))
    S = oracle.covariance(xy, 1.0, 0.05, 0.5, 1e-2)            # short range + nugget: cond ~ 1e2
    mu = rng.standard_normal(n)
    obs = np.sort(rng.choice(n, m, replace=False))
    y = rng.standard_normal(m)
    Sp, mp = oracle.posterior(S, mu, obs, y, 0.5)
    Sl, ml = oracle.posterior.__globals__["posterior_literal"](S, mu, obs, y, 0.5)
    assert np.linalg.cond(S) < 1e3
    assert np.max(np.abs(Sp - Sl)) <= 1e-12 and np.max(np.abs(mp - ml)) <= 1e-12


def test_independent_block_unchanged_and_limits():
    S = np.diag([1.0, 2.0, 3.0])
    Sp, mp = oracle.posterior(S, np.zeros(3), np.array([1]), np.array([0.7]), 0.5)
    assert Sp[0, 0] == pytest.approx(1.0) and Sp[2, 2] == pytest.approx(3.0) and mp[0] == 0 and mp[2] == 0
    # tiny noise: the observed site collapses onto its observation
    Sp, mp = oracle.posterior(S, np.zeros(3), np.array([1]), np.array([0.7]), 1e-5)
    assert mp[1] == pytest.approx(0.7, rel=1e-9) and Sp[1, 1] < 1e-9
    # huge noise: no information
    Sp, mp = oracle.posterior(S, np.zeros(3), np.array([1]), np.array([0.7]), 1e5)
    assert np.allclose(Sp, S, atol=1e-9) and np.allclose(mp, 0, atol=1e-9)


def test_crd_cov_reduces_to_crd_for_the_prior():
    """Alg. 1 on a given covariance (crd_cov, used for Sigma_post) equals Alg. 1 built from the
    locations (crd) when the covariance is the prior Matérn one."""
    import workloads as W
    cfg = W.small_config("cov-pin", 8, 500, 2)
    inp = W.make_inputs(cfg)
    S = oracle.covariance(inp.xy, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget)
    r1 = oracle.crd(inp.xy, inp.mu, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget, cfg.u, cfg.N, cfg.R, cfg.seed_lattice,
                    cfg.conf)
    r2 = oracle.crd_cov(S, inp.mu, cfg.u, cfg.N, cfg.R, cfg.seed_lattice, cfg.conf)
    assert np.array_equal(r1.order, r2.order)
    assert np.max(np.abs(r1.logp - r2.logp)) <= 1e-13
    assert np.array_equal(r1.k_star, r2.k_star)
