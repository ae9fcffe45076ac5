"""CPU-only checks of the C ABI library: it loads, exports every symbol include/mvn.h declares, and
its host-side steps (lattice tables, marginal order, regions) agree bit for bit with the oracle.
No compute is issued to a GPU here."""
import math
import re
import os

import numpy as np
import pytest

import oracle
from oracle import lattice
import paper_2405_14892_b200 as mvn

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "mvn.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mvn_[a-z_]+)\s*\(", src)))


def test_header_symbols_exported():
    decl = header_functions()
    assert sorted(mvn.ABI_SYMBOLS) == decl
    L = mvn.lib()
    for name in decl:
        assert hasattr(L, name), name
    assert b"sm_100a" in L.mvn_version()


def test_create_fails_loudly_without_b200():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    h = __import__("ctypes").c_void_p()
    st = mvn.lib().mvn_create(0, None, __import__("ctypes").byref(h))
    assert st == mvn.MVN_E_CUDA


def test_tile_sizes():
    assert mvn.mvn_tiles_count(1) == 1
    assert mvn.mvn_tiles_count(128) == 1
    assert mvn.mvn_tiles_count(129) == 3
    assert mvn.mvn_tiles_bytes(400) == 10 * 128 * 128 * 8
    assert mvn.mvn_tiles_bytes(65536) == 512 * 513 // 2 * 128 * 128 * 8   # 17.2 GB (config D)
    bad = mvn.mvn_tiles(100, 64)
    assert mvn.lib().mvn_tiles_count(bad) == -1


def test_lattice_generators_bitwise_vs_oracle():
    n = 102_400                                   # config E
    g = mvn.mvn_lattice_generators(n)
    assert np.array_equal(g, lattice.generators(n))


def test_lattice_shifts_bitwise_vs_oracle():
    for seed, R, n in [(3001, 10, 400), (0, 1, 5), (2 ** 64 - 1, 3, 1000)]:
        assert np.array_equal(mvn.mvn_lattice_shifts(seed, R, n), lattice.shifts(seed, R, n))


def test_marginal_order_bitwise_vs_oracle():
    import workloads as W
    for name in ("A", "B"):
        inp = W.make_inputs(name)
        c = inp.cfg
        var = np.full(c.n, c.sigma2 + c.nugget)
        o1, a1, p1 = mvn.mvn_marginal_order(inp.mu, var, c.u)
        o2, a2, p2 = oracle.marginal_order(inp.mu, var, c.u)
        assert np.array_equal(o1, o2)
        assert np.array_equal(a1, a2)
        assert np.max(np.abs(p1 - p2)) <= 2e-16
    mu = np.array([0.5, 1.0, 0.5, -2.0, 1.0])
    o, a, _ = mvn.mvn_marginal_order(mu, np.ones(5), 0.2)
    assert list(o) == [1, 4, 0, 2, 3]
    with pytest.raises(mvn.MvnError):
        mvn.mvn_marginal_order(np.array([np.nan]), np.ones(1), 0.0)
    with pytest.raises(mvn.MvnError):
        mvn.mvn_marginal_order(np.array([0.0]), np.zeros(1), 0.0)


def test_confidence_region_vs_oracle():
    rng = np.random.default_rng(0)
    for trial in range(50):
        n = int(rng.integers(0, 300))
        lp = -np.cumsum(rng.exponential(0.01, n))
        if n and trial % 3 == 0:
            lp[rng.integers(0, n)] += 1e-3            # non-monotone input: running min applies
        conf = [t / 100 for t in range(50, 100)]
        k1, t1 = mvn.mvn_confidence_region(lp, conf)
        k2, t2 = oracle.region(lp, conf)
        assert np.array_equal(k1, k2)
        assert np.array_equal(t1, t2)
    with pytest.raises(mvn.MvnError):
        mvn.mvn_confidence_region(np.array([-0.1]), [1.0])
    with pytest.raises(mvn.MvnError):
        mvn.mvn_confidence_region(np.array([np.nan]), [0.5])


def test_prefix_shift_stats_vs_oracle():
    """mvn_prefix_shift_stats (host C) against oracle.shift_stats: random per-shift estimates, a row
    far below the double range, an exactly equal row (rel_se 0), an all -inf row (NaN), R = 1."""
    rng = np.random.default_rng(4)
    R, n = 8, 50
    L = np.cumsum(-rng.uniform(0.0, 0.2, (1, n)), axis=1) + rng.normal(0, 0.05, (R, n))
    L[:, 10] -= 1000.0
    L[:, 11] = -3.25
    L[:, 12] = -np.inf
    lp, se = mvn.mvn_prefix_shift_stats(L)
    lpo, seo = oracle.shift_stats(L)
    fin = np.isfinite(lpo)
    assert np.array_equal(fin, np.isfinite(lp))
    assert np.max(np.abs(lp[fin] - lpo[fin])) <= 1e-13
    assert np.max(np.abs(se[fin] - seo[fin])) <= 1e-13
    assert se[11] == 0.0 and np.isnan(se[12]) and lp[12] == -np.inf
    lp1, se1 = mvn.mvn_prefix_shift_stats(L[:1])
    assert np.array_equal(lp1[fin], L[0][fin]) and np.all(se1[fin] == 0.0)
