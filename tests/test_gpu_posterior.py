"""NEXT-4 on the GPU: posterior conditioning (Eq. 7-8) through mvn_posterior / mvn_posterior_tiles
against the oracle (oracle/posterior.py: Eq. 7-8 literally, dense inverses), and Alg. 1 on the
posterior field (mvn.crd_posterior vs oracle.crd_cov). Tolerances: mu_post and Sigma_post within
1e-11 (the oracle's push-through solve and the GPU's Cholesky of Sigma_oo + tau^2 I are both
well conditioned, cond <= 1 + lambda_max/tau^2); log P_k within the north_star 1e-8, identical
order and regions."""
import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch(cuda_device):
    import torch as t
    return t


def mvn():
    import paper_2405_14892_b200 as m
    return m


def dense(T, n):
    return mvn().mvn_unpack_lower(T, n).T.contiguous().cpu().numpy()


@pytest.mark.parametrize("g,m,base", [(20, 60, "A"), (23, 300, "C"), (12, 1, "A"), (15, 128, "A"), (16, 256, "B")])
def test_posterior_vs_oracle(torch, g, m, base):
    cfg = W.small_config(f"post{g}", g, 500, 2, base=base)
    P = W.make_posterior_inputs(cfg, m)
    mp, vp = mvn().mvn_posterior(P.xy, P.mu, P.obs, P.y, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget, P.tau)
    Sp, mpo = oracle.posterior_field(P.xy, P.mu, P.obs, P.y, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget, P.tau)
    assert np.max(np.abs(mp - mpo)) <= 1e-11
    assert np.max(np.abs(vp - np.diag(Sp))) <= 1e-11
    order, a, _ = mvn().mvn_marginal_order(mp, vp, cfg.u)
    T = mvn().mvn_posterior_tiles(order)
    G = dense(T, cfg.n)
    want = np.tril(Sp[np.ix_(order, order)])
    assert np.max(np.abs(G - want)) <= 1e-11


def test_crd_on_posterior_vs_oracle(torch):
    cfg = W.small_config("postcrd", 20, 2000, 4, base="A")
    P = W.make_posterior_inputs(cfg, 70)
    out, mp, vp, _ = mvn().crd_posterior(P.xy, P.mu, P.obs, P.y, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget, P.tau,
                                         cfg.u, cfg.N, cfg.R, cfg.seed_lattice, cfg.conf)
    Sp, mpo = oracle.posterior_field(P.xy, P.mu, P.obs, P.y, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget, P.tau)
    ref = oracle.crd_cov(Sp, mpo, cfg.u, cfg.N, cfg.R, cfg.seed_lattice, cfg.conf, chunk=500, nthreads=16)
    assert out.info == -1
    assert np.array_equal(out.order, ref.order)
    assert np.max(np.abs(out.logP - ref.logp)) <= 1e-8
    assert np.array_equal(out.k_star, ref.k_star)
    # the observations move the field: the posterior regions differ from the prior marginal picture
    assert not np.allclose(mp, 0.0)


def test_posterior_argument_errors(torch):
    xy = np.random.default_rng(0).uniform(size=(50, 2))
    with pytest.raises(mvn().MvnError):
        mvn().mvn_posterior(xy, np.zeros(50), np.array([3, 3]), np.zeros(2), 1.0, 0.1, 0.5, 1e-8, 0.5)
    with pytest.raises(mvn().MvnError):
        mvn().mvn_posterior(xy, np.zeros(50), np.array([3]), np.zeros(1), 1.0, 0.1, 0.5, 1e-8, 0.0)
    with pytest.raises(mvn().MvnError):
        mvn().mvn_posterior(xy, np.zeros(50), np.array([50]), np.zeros(1), 1.0, 0.1, 0.5, 1e-8, 0.5)
