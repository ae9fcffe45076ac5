"""Pins of the oracle's special functions, lattice and Matérn against what mathematics fixes
(closed forms, mpmath at 50 digits, published test vectors). CPU only."""
import math
from decimal import Decimal, getcontext
from fractions import Fraction

import mpmath as mp
import numpy as np
import pytest

import oracle
from oracle import lattice

mp.mp.dps = 50


def mp_Phi(x):
    return mp.ncdf(mp.mpf(x))


def mp_bisect(f, lo, hi, iters=220):
    """Root of a monotone f on [lo, hi] by plain bisection (robust; 60-digit arithmetic)."""
    with mp.workdps(60):
        lo, hi = mp.mpf(lo), mp.mpf(hi)
        flo = f(lo)
        for _ in range(iters):
            mid = (lo + hi) / 2
            fm = f(mid)
            if (fm > 0) == (flo > 0):
                lo, flo = mid, fm
            else:
                hi = mid
        return (lo + hi) / 2


def mp_Phiinv(p):
    """Phi^{-1}(p) in 60 digits: bracketed root of log Phi(y) - log p (robust in both tails)."""
    with mp.workdps(60):
        p = mp.mpf(p)
        if p <= 0.5:
            return mp_bisect(lambda y: mp.log(mp.ncdf(y)) - mp.log(p), -45, 0.1)
        return -mp_bisect(lambda y: mp.log(mp.ncdf(y)) - mp.log(1 - p), -45, 0.1)


# ----------------------------------------------------------------------------- Phi / Phi^{-1}
@pytest.mark.parametrize("x", [-37.5, -30.0, -8.0, -1.0, -1e-8, 0.0, 0.3, 1.0, 5.0, 8.0])
def test_Phi_vs_mpmath(x):
    # Phi's condition number is ~x^2 in the tails: the rounding of x/sqrt(2) alone moves Phi by
    # ~x^2 eps relative, so the bound is eps-scaled by (2 + x^2).
    tol = 2.2e-16 * (2 + x * x)
    want = mp_Phi(x)
    got = oracle.Phi(x)
    assert abs(got - float(want)) <= tol * float(want) + 1e-300
    wantb = mp_Phi(-x)
    assert abs(oracle.Phibar(x) - float(wantb)) <= tol * float(wantb) + 1e-300


@pytest.mark.parametrize("p", [1e-300, 1e-200, 1e-50, 1e-17, 1e-8, 0.01, 0.1, 0.3, 0.4999, 0.5])
def test_Phiinv_vs_mpmath(p):
    want = float(mp_Phiinv(p))
    got = oracle.Phiinv(p)
    assert abs(got - want) <= 2e-15 * max(1.0, abs(want))


def test_Phiinv_symmetry_and_roundtrip():
    # round trip on the accurate side of each tail (Phi(x) near 1 has lost the digits of x)
    for x in np.linspace(-37, 0, 75):
        assert abs(oracle.Phiinv(oracle.Phi(x)) - x) <= 1e-14 * max(1, abs(x))
        assert abs(-oracle.Phiinv(oracle.Phibar(-x)) - (-x)) <= 1e-14 * max(1, abs(x))
    assert oracle.Phiinv(0.975) == pytest.approx(1.959963984540054, abs=1e-15)


@pytest.mark.parametrize("z", [24.0, 24.7, 30.0, 100.0, 1e4])
def test_erfcx_far_vs_mpmath(z):
    want = mp.exp(mp.mpf(z) ** 2) * mp.erfc(mp.mpf(z))
    assert abs(oracle.lib().orc_erfcx_far(z) - float(want)) <= 6e-16 * float(want)


@pytest.mark.parametrize("x", [35.0, 37.0, 40.0, 100.0, 1e3])
def test_log_Phibar_far_vs_mpmath(x):
    want = float(mp.log(mp.ncdf(-mp.mpf(x))))
    assert abs(oracle.lib().orc_log_Phibar_far(x) - want) <= 2e-16 * abs(want)


@pytest.mark.parametrize("x0,delta", [(35.0, 0.0), (40.0, -1.0), (40.0, -30.0), (36.0, -200.0)])
def test_Phibar_inv_far_solves(x0, delta):
    T = float(mp.log(mp.ncdf(-mp.mpf(x0)))) + delta
    y = oracle.lib().orc_Phibar_inv_far(T, x0)
    want = float(mp_bisect(lambda t: mp.log(mp.ncdf(-t)) - T, 30, 100))
    assert abs(y - want) <= 4e-16 * want


# ----------------------------------------------------------------------------- one SOV step (R9)
def mp_step(ap, bp, w):
    """Eq. 2-3 evaluated at 60 digits: q = Phi(b') - Phi(a'), y = Phi^{-1}(Phi(a') + w q)."""
    with mp.workdps(60):
        A = mp.mpf(0) if ap == -math.inf else mp.ncdf(mp.mpf(ap))
        B = mp.mpf(1) if bp == math.inf else mp.ncdf(mp.mpf(bp))
        # use upper tails when far right, to keep digits
        Ab = mp.mpf(1) if ap == -math.inf else mp.ncdf(-mp.mpf(ap))
        Bb = mp.mpf(0) if bp == math.inf else mp.ncdf(-mp.mpf(bp))
        q = Ab - Bb if ap > 0 else B - A
        plo = A + mp.mpf(w) * q
        phi = Bb + (1 - mp.mpf(w)) * q
        if plo < phi:
            y = mp_bisect(lambda t: mp.log(mp.ncdf(t)) - mp.log(plo), -100, 100)
        else:
            y = mp_bisect(lambda t: mp.log(mp.ncdf(-t)) - mp.log(phi), -100, 100)
        return float(mp.log(q)), float(y)


W_GRID = [2.0 ** -53, 0.3, 0.5, 0.9, 1 - 2.0 ** -53]


@pytest.mark.parametrize("ap", [-math.inf, -40.0, -8.0, -1.0, 0.0, 0.5, 3.0, 9.6, 30.0, 36.0, 40.0])
@pytest.mark.parametrize("width", [0.1, 5.0, math.inf])
def test_sov_step_vs_mpmath(ap, width):
    bp = ap + width if ap != -math.inf else (width if width != math.inf else math.inf)
    for w in W_GRID:
        lq, y = oracle.sov_step(ap, bp, w)
        wlq, wy = mp_step(ap, bp, w)
        assert abs(lq - wlq) <= 1e-14 * max(1.0, abs(wlq)), (ap, bp, w, lq, wlq)
        assert abs(y - wy) <= 1e-13 * max(1.0, abs(wy)), (ap, bp, w, y, wy)
        if bp != math.inf:
            assert ap <= y <= bp or abs(y - ap) < 1e-12 * max(1, abs(ap)) or abs(y - bp) < 1e-12 * max(1, abs(bp))
        else:
            assert y >= ap or ap == -math.inf


def test_sov_step_special_cases():
    # a = -inf, b = +inf: q = 1 exactly, y = Phi^{-1}(w)
    for w in W_GRID:
        lq, y = oracle.sov_step(-math.inf, math.inf, w)
        assert lq == 0.0
        assert y == oracle.Phiinv(w) or abs(y - oracle.Phiinv(w)) <= 1e-15 * max(1, abs(y))
    # empty interval
    lq, y = oracle.sov_step(1.0, 1.0, 0.5)
    assert lq == -math.inf and y == 1.0
    # lower far tail by reflection: b' = -40, a' = -inf
    lq, y = oracle.sov_step(-math.inf, -40.0, 0.5)
    assert abs(lq - float(mp.log(mp.ncdf(-40)))) <= 1e-15 * abs(lq)


# ----------------------------------------------------------------------------- lattice (R8)
def test_primes():
    assert lattice.primes(10) == [2, 3, 5, 7, 11, 13, 17, 19, 23, 29]
    assert lattice.primes(10000)[-1] == 104729
    assert lattice.primes(100000)[-1] == 1299709


def test_generators_vs_decimal_sqrt():
    getcontext().prec = 80
    ps = lattice.primes(2000)
    G = lattice.generators(2000)
    for k in list(range(50)) + list(range(1950, 2000)):
        r = Decimal(ps[k]).sqrt()
        frac = r - int(r)
        want = int(frac * (Decimal(2) ** 64))
        assert int(G[k]) == want


def test_splitmix64_published_vectors():
    # SplitMix64 seeded with 0: first three outputs (reference sequence of the generator).
    z = 0
    outs = []
    for _ in range(3):
        z = (z + lattice.GAMMA) & lattice.MASK64
        outs.append(lattice.splitmix64_mix(z))
    assert outs == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    D = lattice.shifts(0, 1, 1)
    assert int(D[0, 0]) == 0xE220A8397B1DCDAF


def test_w_exact_and_in_unit_interval():
    G = lattice.generators(16)
    D = lattice.shifts(3001, 2, 16)
    for k in range(16):
        for j in (1, 2, 777, 10_000, 2 ** 40):
            w = oracle.lib().orc_lattice_w(j, int(G[k]), int(D[1, k]))
            assert w == lattice.lattice_w(j, G[k], D[1, k])
            f = Fraction(w)
            assert 0 < f < 1
            assert f.denominator == 2 ** 53            # odd multiple of 2^-53
            assert Fraction(1.0 - w) == 1 - f          # 1 - w exact in fp64


def test_lattice_integration_converges_like_qmc():
    # 1-D rank-1 lattice frac(j sqrt2 + D): error of a smooth integral is O(log N / N) (bounded
    # partial quotients of sqrt 2), far below the MC rate 1/sqrt(N).
    G = int(lattice.generators(1)[0])
    D = int(lattice.shifts(7, 1, 1)[0, 0])
    for N in (1000, 10000, 100000):
        w = np.array([lattice.lattice_w(j, G, D) for j in range(1, N + 1)])
        err = abs(np.mean(w * w) - 1.0 / 3.0)
        assert err <= 3.0 * math.log(N) / N


# ----------------------------------------------------------------------------- Matérn (Eq. 6)
def test_matern_closed_forms():
    x = np.concatenate([[1e-6, 1e-3], np.linspace(0.01, 50, 200)])
    beta = 0.1
    h = x * beta
    m05 = oracle.matern(h, 1.7, beta, 0.5)
    assert np.max(np.abs(m05 / (1.7 * np.exp(-x)) - 1)) <= 1e-13
    m15 = oracle.matern(h, 1.0, beta, 1.5)
    assert np.max(np.abs(m15 / ((1 + x) * np.exp(-x)) - 1)) <= 1e-13
    m25 = oracle.matern(h, 1.0, beta, 2.5)
    assert np.max(np.abs(m25 / ((1 + x + x * x / 3) * np.exp(-x)) - 1)) <= 1e-13
    assert oracle.matern(np.array([0.0]), 2.5, 0.1, 0.5)[0] == 2.5
    assert oracle.matern(np.array([0.1]), 1.0, 0.1, 0.5)[0] == pytest.approx(math.exp(-1), rel=1e-15)


@pytest.mark.parametrize("nu", [0.3, 1.0, 1.43391, 3.2])
def test_matern_general_nu_vs_mpmath(nu):
    for x in (0.01, 0.5, 2.0, 10.0):
        want = mp.mpf(2) ** (1 - nu) / mp.gamma(nu) * mp.mpf(x) ** nu * mp.besselk(nu, x)
        got = oracle.matern(np.array([x * 0.2]), 1.0, 0.2, nu)[0]
        assert abs(got - float(want)) <= 1e-13 * float(want)
    hs = np.sort(np.random.default_rng(0).uniform(0, 2, 1000))
    v = oracle.matern(hs, 1.0, 0.1, nu)
    assert np.all(np.diff(v) <= 0)


def test_covariance_symmetric_diag():
    xy = np.random.default_rng(1).uniform(size=(50, 2))
    S = oracle.covariance(xy, 1.3, 0.1, 1.5, 1e-8)
    assert np.array_equal(S, S.T)
    assert np.all(np.diag(S) == 1.3 + 1e-8)
    S2 = oracle.covariance(np.array([[0.0, 0.0], [0.1, 0.0]]), 1.0, 0.1, 0.5, 0.0)
    assert S2[1, 0] == pytest.approx(math.exp(-1), rel=1e-15)
