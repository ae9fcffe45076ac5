"""NEXT-4 mixed precision on the SOV GEMM (a6): mvn_sov_prefix_ex with MVN_SOV_INT8 — the update
S = L Y on the int8 tensor cores (tcgen05, 36 exact int8 products of 8-digit splits, reading R24),
the chain and the reductions in fp64 — against the oracle on the same inputs, lattice and shifts
(shared-L mode: the oracle consumes the GPU's L). Bar: the north_star's |dlog P_k| <= 1e-8 for
every prefix (measured ~1e-12 at n = 5,000), identical regions; plus the path's own contract:
b must be +inf, |y| < 63.5 (MVN_E_NUMERIC otherwise), deterministic, range split = one call."""
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


def logp(M, S, NR):
    M, S = M.cpu().numpy(), S.cpu().numpy()
    with np.errstate(divide="ignore"):
        return np.where(S > 0, M + np.log(S) - math.log(NR), -np.inf)


def setup(torch, cfg):
    import test_gpu_parity as P
    inp, order, a = P.sorted_inputs(cfg)
    T = P.gpu_cov(torch, inp.xy[order], cfg)
    assert mvn().mvn_potrf(T, cfg.n) == -1
    return T, a


@pytest.mark.parametrize("base,g,N,R,begin,end", [
    ("A", 9, 300, 2, 0, None),          # n = 81: one row block, no MMA
    ("A", 12, 300, 2, 0, None),         # n = 144: two row blocks, ragged tail
    ("A", 20, 2000, 5, 0, None),        # config A geometry
    ("C", 23, 500, 3, 37, 1_400),       # nu = 3/2, u = 0.5; ragged range across shifts
    ("B", 41, 1000, 2, 0, None),        # n = 1,681
    ("B", 70, 1200, 2, 0, None),        # config B geometry (n = 4,900, 39 row blocks)
])
def test_sov_int8_vs_oracle(torch, base, g, N, R, begin, end):
    import test_gpu_parity as P
    cfg = W.small_config(f"i8{base}{g}", g, N, R, base=base)
    T, a = setup(torch, cfg)
    n = cfg.n
    end = cfg.NR if end is None else end
    d_a = torch.from_numpy(a).cuda()
    M, S = mvn().mvn_sov_prefix_ex(T, n, d_a, cfg.N, cfg.R, cfg.seed_lattice, begin, end, method=INT8)
    lp = logp(M, S, end - begin)
    L = P.to_dense_lower(T, n)
    Mo, So = P.oracle_range(L, a, np.full(n, np.inf), cfg.N, cfg.R, cfg.seed_lattice, begin, end)
    lo = P.logp_from(Mo, So, end - begin)
    d = float(np.max(np.abs(lp - lo)))
    assert d <= 1e-8, d
    assert d <= 1e-10, d                    # measured ~1e-12 at these sizes
    k, _ = mvn().mvn_confidence_region(lp, cfg.conf)
    ko, tie = oracle.region(lo, cfg.conf)
    assert all(x == y or t for x, y, t in zip(k, ko, tie))


def test_sov_int8_contract(torch):
    cfg = W.small_config("i8c", 15, 400, 2, base="A")
    T, a = setup(torch, cfg)
    n = cfg.n
    d_a = torch.from_numpy(a).cuda()
    M1, S1 = mvn().mvn_sov_prefix_ex(T, n, d_a, cfg.N, cfg.R, 9, method=INT8)
    M2, S2 = mvn().mvn_sov_prefix_ex(T, n, d_a, cfg.N, cfg.R, 9, method=INT8)
    assert torch.equal(M1, M2) and torch.equal(S1, S2)                       # deterministic
    # the multi-GPU combine on one device: two ranges, rescaled and summed == one call
    Ma, Sa = mvn().mvn_sov_prefix_ex(T, n, d_a, cfg.N, cfg.R, 9, 0, 333, method=INT8)
    Mb, Sb = mvn().mvn_sov_prefix_ex(T, n, d_a, cfg.N, cfg.R, 9, 333, cfg.NR, method=INT8)
    Mg = torch.maximum(Ma, Mb)
    mvn().mvn_prefix_rescale(Mg, Ma, Sa)
    mvn().mvn_prefix_rescale(Mg, Mb, Sb)
    lp_split = mvn().mvn_prefix_finalize(Mg, Sa + Sb, cfg.NR).cpu().numpy()
    lp_one = mvn().mvn_prefix_finalize(M1, S1, cfg.NR).cpu().numpy()
    assert np.max(np.abs(lp_split - lp_one)) <= 1e-12
    with pytest.raises(mvn().MvnError):                                      # finite b: fp64 path only
        mvn().mvn_sov_prefix_ex(T, n, d_a, cfg.N, cfg.R, 9, b=d_a + 1.0, method=INT8)
    with pytest.raises(mvn().MvnError):
        mvn().mvn_sov_prefix_ex(T, n, d_a, cfg.N, cfg.R, 9, method=7)


def test_sov_int8_y_out_of_range(torch):
    """Sigma = I with a = 70: every y ~ 70 lies outside the int8 path's fixed scale (|y| < 63.5):
    MVN_E_NUMERIC, not a wrong answer; a = 30 (y ~ 30) stays inside and matches the closed form
    k log Phibar(30)."""
    from scipy.special import log_ndtr
    n = 200
    T = mvn().mvn_pack_lower(torch.from_numpy(np.eye(n)).cuda(), n)
    mvn().mvn_potrf(T, n)
    with pytest.raises(mvn().MvnError) as e:
        mvn().mvn_sov_prefix_ex(T, n, torch.full((n,), 70.0, dtype=torch.float64, device="cuda"), 128, 2, 3,
                                method=INT8)
    assert e.value.status == mvn().MVN_E_NUMERIC
    M, S = mvn().mvn_sov_prefix_ex(T, n, torch.full((n,), 30.0, dtype=torch.float64, device="cuda"), 128, 2, 3,
                                   method=INT8)
    lp = logp(M, S, 256)
    want = np.arange(1, n + 1) * log_ndtr(-30.0)
    # s = 0 exactly (Sigma = I): what remains is the device log Phibar(30) against scipy's, a fixed
    # relative bias (measured 4.2e-15) that adds up over the 200 identical rows
    assert np.all(np.abs(lp - want) <= 1e-12 + 1e-14 * np.abs(want))


@pytest.mark.parametrize("method", [1, 3])
def test_mvn_crd_mixed_precision_vs_oracle(torch, monkeypatch, method):
    """The public end-to-end C call with the mixed-precision bits (1: int8 SOV GEMM, 3: and the int8
    Cholesky updates, forced on at this size) on config B's geometry: the north_star bars against
    the oracle's own pipeline (independent mode): |dlog P| <= 1e-8, identical order and regions."""
    monkeypatch.setenv("MVN_POTRF_OZ_ALWAYS", "1")
    cfg = W.small_config("crd8", 50, 2000, 4, base="B")
    inp = W.make_inputs(cfg)
    out = mvn().mvn_crd(inp.xy, inp.mu, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget, cfg.u, cfg.N, cfg.R,
                        cfg.seed_lattice, cfg.conf, method=method)
    ref = oracle.crd(inp.xy, inp.mu, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget, cfg.u, cfg.N, cfg.R,
                     cfg.seed_lattice, cfg.conf, chunk=1000, nthreads=0)
    assert out.info == -1
    assert np.array_equal(out.order, ref.order)
    assert np.max(np.abs(out.logP - ref.logp)) <= 1e-8
    assert np.array_equal(out.k_star, ref.k_star)
