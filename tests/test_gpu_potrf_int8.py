"""NEXT-4 mixed precision on the Cholesky (a3): mvn_potrf_ex with MVN_POTRF_INT8 — the trailing
updates on the int8 tensor cores (reading R25), the panel work on fp64 DMMA — against the oracle:
residual ||L L^T - Sigma||_F / ||Sigma||_F <= 1e-12 (north_star), elementwise within the fp64
factor's conditioning bound, the failing row of a non-SPD matrix, and the whole pipeline (int8 factor
+ SOV) against the oracle's own factor within the north_star 1e-8 on log P."""
import math

import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu
INT8 = 1


@pytest.fixture(scope="module")
def torch(cuda_device):
    import torch as t
    return t


def mvn():
    import paper_2405_14892_b200 as m
    return m


@pytest.fixture
def always_int8(monkeypatch):
    """Every trailing update on the int8 path (by default only kp = 8 super-panels with >= 4 tiles
    per cluster take it, i.e. n >= 49,152)."""
    monkeypatch.setenv("MVN_POTRF_OZ_ALWAYS", "1")


@pytest.mark.parametrize("n,nu", [(300, 0.5), (2000, 1.5), (5000, 0.5), (9000, 0.5), (13 * 128 + 5, 1.5)])
def test_potrf_int8_vs_oracle(torch, always_int8, n, nu):
    import test_gpu_parity as P
    xy = np.random.default_rng(100 + n).uniform(size=(n, 2))
    beta = 0.1 if nu == 0.5 else 0.05
    T = mvn().mvn_cov_matern(torch.from_numpy(xy).cuda(), 1.0, beta, nu, 1e-8)
    R = T.clone()
    assert mvn().mvn_potrf_ex(T, n, INT8) == -1
    assert mvn().mvn_potrf(R, n) == -1
    Lg = P.to_dense_lower(T, n)
    S = oracle.covariance(xy, 1.0, beta, nu, 1e-8)
    res = np.linalg.norm(Lg @ Lg.T - S) / np.linalg.norm(S)
    assert res <= 1e-12, res
    Lo, info = oracle.cholesky(S, nthreads=8)
    cond = np.linalg.cond(S)
    assert np.max(np.abs(Lg - Lo)) <= max(1e-13, 50 * cond * 2.2e-16)
    d = float((T - R).abs().max())
    assert d <= max(1e-13, 50 * cond * 2.2e-16), d                  # vs the fp64 DMMA factor


def test_potrf_int8_not_spd_reports_row(torch, always_int8):
    n = 1200
    A = np.eye(n)
    A[777, 777] = -1.0
    T = mvn().mvn_pack_lower(torch.from_numpy(A).cuda(), n)
    assert mvn().mvn_potrf_ex(T, n, INT8, raise_on_numeric=False) == 777


def test_pipeline_int8_factor_vs_oracle(torch, always_int8):
    """Config B geometry end to end with the int8 factor (independent mode: the oracle factors Sigma
    itself) and both SOV arithmetics: |dlog P| <= 1e-8, identical regions."""
    cfg = W.small_config("Bp8", 70, 2000, 4, base="B")
    inp = W.make_inputs(cfg)
    n = cfg.n
    ref = oracle.crd(inp.xy, inp.mu, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget, cfg.u, cfg.N, cfg.R,
                     cfg.seed_lattice, cfg.conf, chunk=1000, nthreads=0)
    order, a, _ = mvn().mvn_marginal_order(inp.mu, np.full(n, cfg.sigma2 + cfg.nugget), cfg.u)
    assert np.array_equal(order, ref.order)
    d_xy = torch.from_numpy(np.ascontiguousarray(inp.xy[order])).cuda()
    d_a = torch.from_numpy(a).cuda()
    T = mvn().mvn_cov_matern(d_xy, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget)
    assert mvn().mvn_potrf_ex(T, n, INT8) == -1
    for method in (0, 1):
        M, S = mvn().mvn_sov_prefix_ex(T, n, d_a, cfg.N, cfg.R, cfg.seed_lattice, method=method)
        lp = mvn().mvn_prefix_finalize(M, S, cfg.NR).cpu().numpy()
        assert np.max(np.abs(lp - ref.logp)) <= 1e-8
        k, _ = mvn().mvn_confidence_region(lp, cfg.conf)
        assert np.array_equal(k, ref.k_star)


@pytest.mark.slow
def test_potrf_int8_default_threshold_large(torch):
    """n = 51,277 (kp = 8: the default int8 regime): against the fp64 DMMA factor elementwise and the
    residual on 2,000 sampled entries (L L^T)_ij vs the oracle's Matern Sigma_ij."""
    import test_gpu_parity as P
    n = 400 * 128 + 77
    xy = np.random.default_rng(9).uniform(size=(n, 2))
    T = mvn().mvn_cov_matern(torch.from_numpy(xy).cuda(), 1.0, 0.03, 0.5, 1e-8)
    R = T.clone()
    assert mvn().mvn_potrf_ex(T, n, INT8) == -1
    assert mvn().mvn_potrf(R, n) == -1
    assert float((T - R).abs().max()) <= 1e-12
    rng = np.random.default_rng(5)
    ii = np.sort(rng.integers(0, n, 2000))
    jj = np.array([rng.integers(0, i + 1) for i in ii])
    got = np.einsum("ij,ij->i", P.tile_rows(T, n, ii, n), P.tile_rows(T, n, jj, n))
    h = np.sqrt(((xy[ii] - xy[jj]) ** 2).sum(1))
    want = oracle.matern(h, 1.0, 0.03, 0.5) + np.where(ii == jj, 1e-8, 0.0)
    assert np.max(np.abs(got - want)) <= 1e-12
