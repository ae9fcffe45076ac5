"""Pins of the oracle's NEXT-2 Monte-Carlo validation (oracle/mcval.py, orc_mc_first) against what
the mathematics fixes: the z generator (SplitMix64 counters vs Python integers, Phi^{-1} vs
mpmath, N(0,1) moments and a KS test), the first-failing-row logic vs a numpy brute force,
closed forms (identity Sigma: product of marginals; equicorrelated rho = 1/2 orthant prefixes
P_k = 1/(k+1); n = 1), and cross-oracle agreement with the QMC sweep. CPU only."""
import math

import mpmath as mp
import numpy as np
import pytest
from scipy import stats
from scipy.special import ndtr

import oracle
from oracle import lattice


def test_mc_mix_matches_python_integers():
    for seed, s, k in [(0, 0, 0), (1234, 5, 77), (2**63 + 11, 49_999, 102_399), (99, 2**20, 3)]:
        want = lattice.splitmix64_mix(seed + lattice.GAMMA * ((s << 32) + k + 1))
        assert oracle.lib().orc_mc_mix(seed, s, k) == want


def test_mc_z_vs_mpmath():
    mp.mp.dps = 40
    for seed, s, k in [(7, 0, 0), (7, 1, 0), (7, 0, 1), (3, 12345, 678), (11, 2, 9), (5, 40_000, 65_000)]:
        X = lattice.splitmix64_mix(seed + lattice.GAMMA * ((s << 32) + k + 1))
        w = mp.mpf((X >> 12)) * mp.mpf(2) ** -52 + mp.mpf(2) ** -53
        want = float(mp.sqrt(2) * mp.erfinv(2 * w - 1))
        assert oracle.mc_z(seed, s, k) == pytest.approx(want, rel=2e-15, abs=1e-300)


def test_mc_z_is_standard_normal():
    z = np.array([oracle.mc_z(17, s, k) for s in range(2000) for k in range(20)])
    n = z.size
    assert abs(z.mean()) <= 4 / math.sqrt(n)
    assert abs(z.var() - 1) <= 4 * math.sqrt(2 / n)
    assert stats.kstest(z, "norm").pvalue > 1e-3


def test_first_failing_row_vs_numpy_bruteforce():
    rng = np.random.default_rng(5)
    n, ns, seed = 12, 3000, 21
    A = rng.standard_normal((n, n))
    S = A @ A.T / n + np.eye(n)
    L = np.linalg.cholesky(S)
    a = rng.uniform(-1.5, 0.3, n)
    f = oracle.mc_first(L, a, seed, 100, ns)
    Z = np.array([[oracle.mc_z(seed, 100 + s, k) for k in range(n)] for s in range(ns)])
    X = Z @ L.T
    bad = X <= a
    want = np.where(bad.any(axis=1), bad.argmax(axis=1), n)
    assert np.array_equal(f, want)


def se_binom(p, N):
    return math.sqrt(max(p * (1 - p), 1e-12) / N)


def test_identity_sigma_product_of_marginals():
    n, N = 6, 40_000
    a = np.array([-1.0, -0.5, -2.0, 0.0, -1.2, -0.3])
    f = oracle.mc_first(np.eye(n), a, 3, 0, N)
    ph = oracle.mc_levels(oracle.mc_counts(f, n), range(n + 1), N)
    assert ph[0] == 1.0
    for k in range(1, n + 1):
        p = float(np.prod(1 - ndtr(a[:k])))
        assert abs(ph[k] - p) <= 4 * se_binom(p, N), (k, ph[k], p)
    assert np.all(np.diff(ph) <= 0)


def test_n1_closed_form():
    N = 50_000
    for a0, s in [(0.0, 1.0), (-0.7, 2.0), (1.1, 0.5)]:
        f = oracle.mc_first(np.array([[s]]), np.array([a0]), 9, 0, N)
        p = 1 - ndtr(a0 / s)
        assert abs(np.mean(f >= 1) - p) <= 4 * se_binom(p, N)


def test_equicorrelated_orthant_prefixes():
    n, N, rho = 10, 40_000, 0.5
    S = (1 - rho) * np.eye(n) + rho * np.ones((n, n))
    L = np.linalg.cholesky(S)
    f = oracle.mc_first(L, np.zeros(n), 4, 0, N)
    ph = oracle.mc_levels(oracle.mc_counts(f, n), range(1, n + 1), N)
    for k in range(1, n + 1):
        p = 1 / (k + 1)
        assert abs(ph[k - 1] - p) <= 4 * se_binom(p, N), (k, ph[k - 1], p)


def test_mc_agrees_with_qmc_sweep():
    """The MC estimate of every prefix and the QMC sweep agree within 4 combined standard errors
    on a config-A-like problem (n = 100 sorted locations, nu = 1/2)."""
    import workloads as W
    cfg = W.small_config("mc-pin", 10, 2000, 5)
    inp = W.make_inputs(cfg)
    var = np.full(cfg.n, cfg.sigma2 + cfg.nugget)
    order, a, _ = oracle.marginal_order(inp.mu, var, cfg.u)
    S = oracle.covariance(inp.xy[order], cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget)
    L, info = oracle.cholesky(S)
    assert info == -1
    N = 40_000
    f = oracle.mc_first(L, a, 77, 0, N, nthreads=8)
    ph = oracle.mc_levels(oracle.mc_counts(f, cfg.n), range(1, cfg.n + 1), N)
    G, D = lattice.generators(cfg.n), lattice.shifts(cfg.seed_lattice, cfg.R, cfg.n)
    parts = oracle.sov_units(L, a, np.full(cfg.n, np.inf), G, D, cfg.N, cfg.R, cfg.N)
    M, Ssum = oracle.combine_units(parts)
    P = np.exp(oracle.prefix_logp(M, Ssum, cfg.NR))
    sq = np.std(np.exp(oracle.per_shift_logp(parts, cfg.N, cfg.R, cfg.N)), axis=0, ddof=1) / math.sqrt(cfg.R)
    for k in range(cfg.n):
        tol = 4 * math.hypot(se_binom(P[k], N), sq[k]) + 1e-4
        assert abs(ph[k] - P[k]) <= tol, (k, ph[k], P[k])


def test_levels_from_counts():
    count = np.array([3, 0, 2, 5])          # n = 3: f in {0, 1, 2, 3}
    assert list(oracle.mc_levels(count, [0, 1, 2, 3], 10)) == [1.0, 0.7, 0.7, 0.5]
