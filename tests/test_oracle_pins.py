"""Pins of the oracle's Cholesky, SOV/QMC sweep, prefix estimator and regions against what the
paper and the mathematics fix: closed forms (n = 1, diagonal Sigma, bivariate / trivariate
orthants, equicorrelated prefixes P_k = 1/(k+1)), AR(1) Cholesky, brute-force Monte Carlo, the
Alg. 1 prefix-collapse identity (R1), and region invariants. CPU only."""
import math

import mpmath as mp
import numpy as np
import pytest
from scipy import integrate
from scipy.special import ndtr

import oracle
from oracle import lattice

INF = math.inf


def run_sov(L, a, b, N, R, seed, chunk=None):
    n = L.shape[0]
    G = lattice.generators(n)
    D = lattice.shifts(seed, R, n)
    chunk = chunk or N
    parts = oracle.sov_units(L, a, b, G, D, N, R, chunk)
    M, S = oracle.combine_units(parts)
    logp = oracle.prefix_logp(M, S, N * R)
    lps = oracle.per_shift_logp(parts, N, R, chunk)
    P = np.exp(logp)
    se = np.std(np.exp(lps), axis=0, ddof=1) / math.sqrt(R)
    return logp, P, se


# ----------------------------------------------------------------------------- Cholesky
def test_cholesky_small_closed_forms():
    L, info = oracle.cholesky(np.eye(5))
    assert info == -1 and np.array_equal(L, np.eye(5))
    L, info = oracle.cholesky(np.array([[4.0, 2.0], [2.0, 3.0]]))
    assert info == -1
    assert L[0, 0] == 2.0 and L[1, 0] == 1.0 and L[1, 1] == pytest.approx(math.sqrt(2.0), rel=1e-16) and L[0, 1] == 0


def test_cholesky_ar1_closed_form():
    # exponential kernel on a sorted 1-D regular grid = AR(1)/KMS matrix rho^|i-j|:
    # L_i0 = rho^i, L_ij = rho^(i-j) sqrt(1 - rho^2) for j >= 1.
    n, rho = 300, math.exp(-0.1 / 0.3)
    S = oracle.covariance(np.stack([np.arange(n) * 0.1, np.zeros(n)], 1), 1.0, 0.3, 0.5, 0.0)
    L, info = oracle.cholesky(S)
    assert info == -1
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    want = np.where(j == 0, rho ** i, rho ** (i - j) * math.sqrt(1 - rho * rho))
    want = np.where(i >= j, want, 0.0)
    assert np.max(np.abs(L - want)) <= 1e-13


def test_cholesky_residual_matern():
    rng = np.random.default_rng(5)
    xy = rng.uniform(size=(400, 2))
    for nu in (0.5, 1.5):
        S = oracle.covariance(xy, 1.0, 0.1, nu, 1e-8)
        L, info = oracle.cholesky(S, nthreads=4)
        assert info == -1
        res = np.linalg.norm(L @ L.T - S) / np.linalg.norm(S)
        assert res <= 1e-14


def test_cholesky_nonspd_reports_row():
    A = np.array([[1.0, 2.0], [2.0, 1.0]])
    assert oracle.cholesky(A)[1] == 1
    B = np.eye(6)
    B[3, 3] = -1.0
    assert oracle.cholesky(B)[1] == 3
    C = np.eye(4)
    C[2, 2] = np.nan
    assert oracle.cholesky(C)[1] == 2


def test_cholesky_thread_count_invariant():
    xy = np.random.default_rng(9).uniform(size=(200, 2))
    S = oracle.covariance(xy, 1.0, 0.1, 1.5, 1e-8)
    L1, _ = oracle.cholesky(S, nthreads=1)
    L4, _ = oracle.cholesky(S, nthreads=4)
    assert np.array_equal(L1, L4)


# ----------------------------------------------------------------------------- SOV closed forms
@pytest.mark.parametrize("a,sigma", [(0.0, 1.0), (-1.3, 0.7), (2.5, 2.0), (80.0, 2.0), (-INF, 1.0)])
def test_sov_n1_exact(a, sigma):
    # n = 1: every sample gives the same q = Phi(b') - Phi(a'), so P_1 = Phibar(a/sigma) exactly.
    L = np.array([[sigma]])
    logp, _, _ = run_sov(L, np.array([a]), np.array([INF]), 257, 3, 11)
    want = 0.0 if a == -INF else float(mp.log(mp.ncdf(-mp.mpf(a) / sigma)))
    assert abs(logp[0] - want) <= 2e-15 * max(1.0, abs(want))


def test_sov_diagonal_exact():
    # diagonal Sigma: s = 0 always, so ell_k is the same for every sample: product of marginals.
    rng = np.random.default_rng(3)
    n = 12
    sig = rng.uniform(0.5, 2.0, n)
    a = rng.uniform(-2, 1, n)
    b = a + rng.uniform(0.1, 3, n)
    b[::3] = INF
    logp, _, _ = run_sov(np.diag(sig), a, b, 100, 4, 5)
    want = 0.0
    for k in range(n):
        hi = mp.mpf(1) if b[k] == INF else mp.ncdf(mp.mpf(b[k]) / sig[k])
        want += mp.log(hi - mp.ncdf(mp.mpf(a[k]) / sig[k]))
        assert abs(logp[k] - float(want)) <= 1e-13 * max(1, abs(float(want)))


def test_sov_identity_n64_orthant():
    # Sigma = I, a = -inf, b = 0: log P_64 = -64 log 2 (SPEC acceptance, exact up to rounding)
    n = 64
    logp, _, _ = run_sov(np.eye(n), np.full(n, -INF), np.zeros(n), 50, 2, 1)
    assert abs(logp[-1] + 64 * math.log(2)) <= 1e-12
    assert np.allclose(logp, -np.arange(1, n + 1) * math.log(2), rtol=0, atol=1e-12)


@pytest.mark.parametrize("rho", [0.5, -0.3, 0.9])
def test_sov_bivariate_orthant(rho):
    # P(X1 > 0, X2 > 0) = 1/4 + arcsin(rho)/(2 pi)
    L = np.linalg.cholesky(np.array([[1.0, rho], [rho, 1.0]]))
    logp, P, se = run_sov(L, np.zeros(2), np.full(2, INF), 4000, 10, 21)
    want = 0.25 + math.asin(rho) / (2 * math.pi)
    assert abs(P[1] - want) <= 3 * se[1] + 1e-12
    assert abs(P[0] - 0.5) <= 1e-15


def test_sov_bivariate_rectangle_vs_quadrature():
    rho, s1, s2 = 0.6, 1.3, 0.8
    Sig = np.array([[s1 * s1, rho * s1 * s2], [rho * s1 * s2, s2 * s2]])
    L = np.linalg.cholesky(Sig)
    a = np.array([-0.4, 0.2])
    b = np.array([1.5, INF])
    logp, P, se = run_sov(L, a, b, 4000, 10, 8)
    # P(a1 < X1 < b1, X2 > a2) = int_{a1/s1}^{b1/s1} phi(z) Phibar((a2/s2 - rho z)/sqrt(1-rho^2)) dz
    f = lambda z: math.exp(-z * z / 2) / math.sqrt(2 * math.pi) * ndtr(-(a[1] / s2 - rho * z) / math.sqrt(1 - rho * rho))
    want, _ = integrate.quad(f, a[0] / s1, b[0] / s1, epsabs=1e-14, epsrel=1e-13)
    assert abs(P[1] - want) <= 3 * se[1] + 1e-12


def test_sov_trivariate_orthants():
    # equicorrelated rho = 1/2: 1/4 (north_star); general: 1/8 + sum arcsin(rho_ij)/(4 pi)
    C = np.full((3, 3), 0.5) + 0.5 * np.eye(3)
    logp, P, se = run_sov(np.linalg.cholesky(C), np.zeros(3), np.full(3, INF), 4000, 10, 2)
    assert abs(P[2] - 0.25) <= 3 * se[2] + 1e-12
    C = np.array([[1.0, 0.3, -0.2], [0.3, 1.0, 0.6], [-0.2, 0.6, 1.0]])
    logp, P, se = run_sov(np.linalg.cholesky(C), np.zeros(3), np.full(3, INF), 4000, 10, 3)
    want = 0.125 + (math.asin(0.3) + math.asin(-0.2) + math.asin(0.6)) / (4 * math.pi)
    assert abs(P[2] - want) <= 3 * se[2] + 1e-12


def test_sov_equicorrelated_all_prefixes():
    # Sigma = (1-rho) I + rho 11^T, c = 0, rho = 1/2: P_k = 1/(k+1) for every prefix k.
    # 64 simultaneous comparisons: 4 se (Bonferroni-style for 64 prefixes at ~3 se each).
    n = 64
    C = np.full((n, n), 0.5) + 0.5 * np.eye(n)
    logp, P, se = run_sov(np.linalg.cholesky(C), np.zeros(n), np.full(n, INF), 2000, 10, 4)
    k = np.arange(1, n + 1)
    z = np.abs(P - 1.0 / (k + 1)) / np.maximum(se, 1e-300)
    assert abs(P[0] - 0.5) <= 1e-15
    assert np.all(z[1:] <= 4.0), z.max()


def test_sov_equicorrelated_thresholds_vs_quadrature():
    # general thresholds c_i: P_k = int phi(z) prod_{i<=k} Phibar((c_i - sqrt(rho) z)/sqrt(1-rho)) dz
    n, rho = 20, 0.35
    c = np.sort(np.random.default_rng(4).uniform(-1.0, 0.7, n))
    C = np.full((n, n), rho) + (1 - rho) * np.eye(n)
    logp, P, se = run_sov(np.linalg.cholesky(C), c, np.full(n, INF), 3000, 10, 6)
    for k in (1, 5, 10, 20):
        f = lambda z: math.exp(-z * z / 2) / math.sqrt(2 * math.pi) * np.prod(
            ndtr(-(c[:k] - math.sqrt(rho) * z) / math.sqrt(1 - rho)))
        want, _ = integrate.quad(f, -12, 12, epsabs=1e-15, epsrel=1e-13, limit=200)
        assert abs(P[k - 1] - want) <= 4 * se[k - 1] + 1e-12, (k, P[k - 1], want, se[k - 1])


def test_sov_bruteforce_mc_n5():
    # brute-force Monte Carlo with 10^7 draws on a Matérn Sigma (n = 5): within 3 combined se
    rng = np.random.default_rng(12)
    xy = rng.uniform(size=(5, 2))
    S = oracle.covariance(xy, 1.0, 0.3, 1.5, 1e-8)
    L, _ = oracle.cholesky(S)
    a = np.array([-0.3, -0.1, 0.2, -0.5, 0.0])
    logp, P, se = run_sov(L, a, np.full(5, INF), 4000, 10, 9)
    Nmc = 10_000_000
    cnt = np.zeros(5)
    for _ in range(10):
        x = rng.standard_normal((Nmc // 10, 5)) @ L.T
        ok = np.cumprod(x > a, axis=1)
        cnt += ok.sum(axis=0)
    pmc = cnt / Nmc
    se_mc = np.sqrt(pmc * (1 - pmc) / Nmc)
    assert np.all(np.abs(P - pmc) <= 3 * np.sqrt(se ** 2 + se_mc ** 2) + 1e-12), (P, pmc)


# ----------------------------------------------------------------------------- prefix collapse R1
def test_prefix_collapse_equals_literal_alg1():
    # Alg. 1 l.9-15 as written: one PMVN per prefix k with a = -inf outside the prefix.
    # With Sigma in sorted order, rows after the prefix have q = 1 exactly and never feed back, so
    # the literal call's per-sample log weight equals the sweep's prefix-k weight bit for bit.
    rng = np.random.default_rng(17)
    n, J = 24, 37
    xy = rng.uniform(size=(n, 2))
    S = oracle.covariance(xy, 1.0, 0.2, 1.5, 1e-8)
    L, _ = oracle.cholesky(S)
    a = np.sort(rng.uniform(-1.5, 0.5, n))
    b = np.full(n, INF)
    G = lattice.generators(n)
    D = lattice.shifts(44, 1, n)[0]
    _, ell_sweep, y_sweep = oracle.sov_unit(L, a, b, G, D, 5, J, want_ell=True, want_y=True)
    for k in range(1, n + 1):
        ak = np.where(np.arange(n) < k, a, -INF)
        _, ell_lit, y_lit = oracle.sov_unit(L, ak, b, G, D, 5, J, want_ell=True, want_y=True)
        assert np.array_equal(ell_lit[n - 1], ell_sweep[k - 1])
        assert np.array_equal(y_lit[:k], y_sweep[:k])


def test_unit_split_invariance():
    # the per-prefix estimate does not depend on how samples are grouped into units (beyond rounding)
    rng = np.random.default_rng(2)
    n = 40
    S = oracle.covariance(rng.uniform(size=(n, 2)), 1.0, 0.1, 0.5, 1e-8)
    L, _ = oracle.cholesky(S)
    a = np.sort(rng.uniform(-1, 0.3, n))
    lp1, _, _ = run_sov(L, a, np.full(n, INF), 600, 3, 77, chunk=600)
    lp2, _, _ = run_sov(L, a, np.full(n, INF), 600, 3, 77, chunk=128)
    assert np.max(np.abs(lp1 - lp2)) <= 1e-14 * max(1, np.max(np.abs(lp1)))


def test_monotone_prefixes():
    rng = np.random.default_rng(8)
    n = 60
    S = oracle.covariance(rng.uniform(size=(n, 2)), 1.0, 0.1, 1.5, 1e-8)
    L, _ = oracle.cholesky(S)
    a = np.sort(rng.uniform(-1, 0.5, n))
    lp, _, _ = run_sov(L, a, np.full(n, INF), 500, 2, 5)
    assert np.all(np.diff(lp) <= 0)


# ----------------------------------------------------------------------------- regions (Eq. 4)
def test_region_identity_exact():
    # Sigma = I: P_k = prod of marginals exactly, so k*(c) = largest prefix with product >= c.
    rng = np.random.default_rng(6)
    n = 30
    a = np.sort(rng.uniform(-4.0, -0.5, n))
    lp, _, _ = run_sov(np.eye(n), a, np.full(n, INF), 64, 2, 3)
    conf = [0.5, 0.8, 0.9, 0.95, 0.99]
    ks, ties = oracle.region(lp, conf)
    prod = np.cumsum([float(mp.log(mp.ncdf(-mp.mpf(x)))) for x in a])
    for c, k in zip(conf, ks):
        assert k == int(np.count_nonzero(prod >= math.log(c)))
    assert np.all(np.diff(ks) <= 0)   # nesting: higher confidence -> smaller region


def test_region_nesting_and_joint_within_marginal():
    import workloads as W
    inp = W.make_inputs(W.small_config("A8", 8, 2000, 4))
    c = inp.cfg
    r = oracle.crd(inp.xy, inp.mu, c.sigma2, c.beta, c.nu, c.nugget, c.u, c.N, c.R, c.seed_lattice,
                   [t / 100 for t in range(50, 100)])
    assert np.all(np.diff(r.k_star) <= 0)
    _, _, pM = oracle.marginal_order(inp.mu, np.full(c.n, c.sigma2 + c.nugget), c.u)
    for conf, k in zip([t / 100 for t in range(50, 100)], r.k_star):
        assert k <= np.count_nonzero(pM >= conf)     # joint region within the marginal region


def test_region_edge_cases():
    ks, ties = oracle.region(np.array([-0.01, -0.2, -0.3]), [0.99, 0.5])
    assert list(ks) == [1, 3]                               # log .99 = -0.01005 < -0.01
    ks, _ = oracle.region(np.array([-0.52, -0.2]), [0.6])   # running min guards non-monotone input
    assert ks[0] == 0                                       # exp(-0.52) = 0.5945 < 0.6
    ks, _ = oracle.region(np.array([-0.5, -0.2]), [0.6])
    assert ks[0] == 2
    ks, _ = oracle.region(np.array([]), [0.6])
    assert ks[0] == 0
    ks, ties = oracle.region(np.array([math.log(0.9) + 1e-10]), [0.9])
    assert ks[0] == 1 and ties[0]


def test_marginal_order_ties_and_limits():
    mu = np.array([0.5, 1.0, 0.5, -2.0, 1.0])
    order, a, pM = oracle.marginal_order(mu, np.ones(5), 0.2)
    assert list(order) == [1, 4, 0, 2, 3]          # descending z, ties by ascending index
    assert np.array_equal(a, 0.2 - mu[order])
    assert pM[1] == pytest.approx(ndtr(0.8), rel=1e-15)


# ----------------------------------------------------------------------------- O6 shift statistics
def test_shift_stats_pins():
    """oracle.shift_stats: (1) the combined estimate is the mean over all N R samples
    (equal N per shift), i.e. prefix_logp of the full partials; (2) zero-variance integrands (n = 1,
    diagonal Sigma: every sample gives the same product) have rel_se = 0 exactly; (3) it matches the
    textbook sd / sqrt(R) on P^(r) where P is representable, and stays finite far below the double
    range (log P ~ -1000), where exp(log P^(r)) underflows."""
    rng = np.random.default_rng(3)
    n, N, R = 40, 300, 6
    A = rng.standard_normal((n, n)) * 0.2
    S = A @ A.T + np.eye(n)
    L, _ = oracle.cholesky(S)
    a = rng.normal(-0.3, 0.4, n)
    b = np.full(n, INF)
    G = lattice.generators(n)
    D = lattice.shifts(11, R, n)
    parts = oracle.sov_units(L, a, b, G, D, N, R, N)
    M, Sm = oracle.combine_units(parts)
    full = oracle.prefix_logp(M, Sm, N * R)
    lps = oracle.per_shift_logp(parts, N, R, N)
    logp, rel = oracle.shift_stats(lps)
    assert np.max(np.abs(logp - full)) <= 1e-13
    P = np.exp(lps)
    want = np.std(P, axis=0, ddof=1) / math.sqrt(R) / np.mean(P, axis=0)
    assert np.max(np.abs(rel - want)) <= 1e-12
    assert rel[0] <= 1e-15 and np.all(rel[1:] > 0)       # P_1 = Phibar(a_1 / L_11) for every sample (n = 1)
    # diagonal Sigma: zero variance across shifts
    Ld = np.diag(rng.uniform(0.5, 2.0, n))
    pd = oracle.sov_units(Ld, a, b, G, D, N, R, N)
    _, reld = oracle.shift_stats(oracle.per_shift_logp(pd, N, R, N))
    assert np.max(reld) <= 1e-12
    # far below the double range: the same statistics after a shift of log P by -1000
    logp2, rel2 = oracle.shift_stats(lps - 1000.0)
    assert np.all(np.isfinite(rel2)) and np.max(np.abs(rel2 - rel)) <= 1e-12
    assert np.max(np.abs(logp2 - (logp - 1000.0))) <= 1e-12
