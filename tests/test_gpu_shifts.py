"""Per-shift estimates on the GPU (mvn_sov_prefix_shifts, reading R11) against the
oracle's per-shift estimates on the same L (shared-L mode), and the combined estimate against the
one-sweep mvn_sov_prefix; the relative standard error against oracle.shift_stats."""
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


@pytest.mark.parametrize("base,g,N,R", [("A", 20, 1000, 5), ("B", 23, 700, 3), ("C", 16, 130, 4)])
def test_shift_estimates_vs_oracle(torch, base, g, N, R):
    import test_gpu_parity as P
    cfg = W.small_config("shifts", g, N, R, base=base)
    inp, order, a = P.sorted_inputs(cfg)
    T = P.gpu_cov(torch, inp.xy[order], cfg)
    n = cfg.n
    assert mvn().mvn_potrf(T, n) == -1
    da = torch.from_numpy(a).cuda()
    Ls = mvn().mvn_sov_prefix_shifts(T, n, da, N, R, 17).cpu().numpy()
    Lg = P.to_dense_lower(T, n)
    parts = []
    for r in range(R):
        Mo, So = P.oracle_range(Lg, a, np.full(n, np.inf), N, R, 17, r * N, (r + 1) * N)
        parts.append(P.logp_from(Mo, So, N))
    Lo = np.array(parts)
    assert np.max(np.abs(Ls - Lo)) <= 1e-10
    lp, se = mvn().mvn_prefix_shift_stats(Ls)
    lpo, seo = oracle.shift_stats(Lo)
    assert np.max(np.abs(lp - lpo)) <= 1e-10
    assert np.max(np.abs(se - seo)) <= 1e-8
    M, S = mvn().mvn_sov_prefix(T, n, da, N, R, 17)
    one = P.logp_from(M.cpu().numpy(), S.cpu().numpy(), N * R)
    assert np.max(np.abs(lp - one)) <= 1e-12
    assert se[0] <= 1e-14 and np.all(se[1:] >= 0)


def test_shift_estimates_errors(torch):
    n = 200
    T = mvn().alloc_tiles(n, "cuda")
    a = torch.zeros(n, dtype=torch.float64, device="cuda")
    with pytest.raises(mvn().MvnError):
        mvn().mvn_sov_prefix_shifts(T, n, a, 0, 2, 1)


def test_custom_lattice_generators(torch):
    """mvn_qmc.d_gen: caller-supplied generators G_k replace R8's table; against the
    oracle's sweep with the same G (same shifts), and R8's own table through d_gen = the default."""
    import test_gpu_parity as P
    from oracle import lattice
    cfg = W.small_config("gen", 17, 600, 2, base="B")
    inp, order, a = P.sorted_inputs(cfg)
    T = P.gpu_cov(torch, inp.xy[order], cfg)
    n = cfg.n
    assert mvn().mvn_potrf(T, n) == -1
    da = torch.from_numpy(a).cuda()
    rng = np.random.default_rng(8)
    G = (rng.integers(0, 2 ** 63, n, dtype=np.uint64) * np.uint64(2) + np.uint64(1))      # odd 64-bit generators
    dG = torch.from_numpy(G.view(np.int64)).cuda()
    M, S = mvn().mvn_sov_prefix(T, n, da, cfg.N, cfg.R, 5, gen=dG)
    Lg = P.to_dense_lower(T, n)
    D = lattice.shifts(5, cfg.R, n)
    parts = [oracle.sov_unit(Lg, a, np.full(n, np.inf), G, D[r], 1, cfg.N)[0] for r in range(cfg.R)]
    Mo, So = oracle.combine_units(np.array(parts))
    lg = P.logp_from(M.cpu().numpy(), S.cpu().numpy(), cfg.NR)
    assert np.max(np.abs(lg - P.logp_from(Mo, So, cfg.NR))) <= 1e-10
    G8 = np.array(lattice.generators(n), dtype=np.uint64)
    M8, S8 = mvn().mvn_sov_prefix(T, n, da, cfg.N, cfg.R, 5, gen=torch.from_numpy(G8.view(np.int64)).cuda())
    M0, S0 = mvn().mvn_sov_prefix(T, n, da, cfg.N, cfg.R, 5)
    assert torch.equal(M8, M0) and torch.equal(S8, S0)
    assert np.max(np.abs(lg - P.logp_from(M0.cpu().numpy(), S0.cpu().numpy(), cfg.NR))) > 1e-6   # a different point set
