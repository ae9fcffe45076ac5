"""NEXT-3 on the GPU: the TLR Cholesky (mvn_tlr_potrf, reading R26) against the oracle
(oracle/tlr.py tlr_cholesky: Sigma compressed by LAPACK SVDs, dense Crout per diagonal tile, a
triangular solve and one SVD truncation per L tile).

Bars:
  * exact cases: Sigma = D + F F^T (every tile of Sigma and of L has rank r) gives ranks = r and the
    dense Cholesky factor to 1e-11; eps = 0 gives mvn_potrf's factor;
  * Matérn fields in the sorted order: ranks equal to the oracle's wherever no oracle singular value
    lies within 1e-9 relative of the threshold (a near tie); then L~ within 1e-9 of the oracle's
    (a wrong term or operand moves it by ~eps); the factor slots reproduce the dense tiles;
  * the algorithm's own identity on the GPU result (independent of the oracle): with Sigma~ from
    mvn_tlr_compress, (L~ L~^T - Sigma~)_IJ = (L_IJ - L~_IJ) L_JJ^T has 2-norm < eps ||L_JJ||_2, and
    the diagonal tiles' residual is rounding;
  * SOV on L~ (dense) against the oracle's SOV on the same L~ (shared-L) <= 1e-10, and the
    oracle's whole TLR pipeline (independent) <= 1e-8 in log P when the ranks agree;
  * failing row, rank overflow (kmax) and argument errors."""
import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu
NB = 128


@pytest.fixture(scope="module")
def torch(cuda_device):
    import torch as t
    return t


def mvn():
    import paper_2405_14892_b200 as m
    return m


def dense_lower(T, n):
    return np.tril(mvn().mvn_unpack_lower(T, n).T.contiguous().cpu().numpy())


def dense_sym(T, n):
    L = dense_lower(T, n)
    return L + np.tril(L, -1).T


def sorted_cov(torch, cfg):
    import test_gpu_parity as P
    inp, order, a = P.sorted_inputs(cfg)
    xs = inp.xy[order]
    T = P.gpu_cov(torch, xs, cfg)
    S = oracle.covariance(xs, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget)
    return T, S, a


def near_tie(sig_row, eps, mode, lo, hi):
    if mode == "abs":
        return np.all(np.abs(sig_row[lo:hi] - eps) <= 1e-12 + 2e-6 * eps)   # the QR's dropped R_22 (<= 1e-6 eps)
    return True


def check_slots(f, T, n):
    """U_t V_t^T from the slots equals the dense off-diagonal tile written to T."""
    G = dense_lower(T, n)
    U = f.U.cpu().numpy()
    V = f.V.cpu().numpy()
    r = f.ranks.cpu().numpy()
    nt = -(-n // NB)
    t = 0
    for I in range(1, nt):
        for J in range(I):
            k = int(r[t])
            Ut, Vt = U[t][:k].T, V[t][:k].T          # slot [kmax cols][128 rows] -> 128 x k
            rows = min(NB, n - I * NB)
            P = Ut @ Vt.T
            assert np.max(np.abs(P[:rows] - G[I * NB:I * NB + rows, J * NB:(J + 1) * NB])) <= 1e-14 * max(1.0, np.abs(P).max())
            if k:                                      # V has orthonormal columns
                assert np.max(np.abs(Vt.T @ Vt - np.eye(k))) < 1e-12
            t += 1


def residual_identity(T, Stg, f, eps, n, mode="abs"):
    """(L~ L~^T - Sigma~)_IJ = (L_IJ - L~_IJ) L_JJ^T on the GPU's own result."""
    L = dense_lower(T, n)
    R = L @ L.T - Stg
    nt = -(-n // NB)
    scale = np.max(np.abs(Stg))
    worst = 0.0
    for J in range(nt):
        cJ = slice(J * NB, min((J + 1) * NB, n))
        assert np.max(np.abs(R[cJ, cJ])) < 1e-13 * scale * nt
        nLJJ = np.linalg.norm(L[cJ, cJ], 2)
        for I in range(J + 1, nt):
            rI = slice(I * NB, min((I + 1) * NB, n))
            res = np.linalg.norm(R[rI, cJ], 2)
            if mode == "abs":
                assert res < eps * nLJJ * (1 + 2e-6) + 1e-13 * scale * nt, (I, J, res, eps * nLJJ)
            else:
                assert res <= eps * np.linalg.norm(L[rI, cJ]) * 1.01 * nLJJ + 1e-11 * scale * nt, (I, J, res)
            worst = max(worst, res / (eps * nLJJ) if eps > 0 else res)
    return worst


def test_tlr_potrf_diag_plus_low_rank_exact(torch):
    rng = np.random.default_rng(7)
    n, r = 450, 6
    F = rng.standard_normal((n, r))
    S = F @ F.T + np.diag(rng.uniform(1.0, 3.0, n))
    T = mvn().mvn_pack_lower(torch.from_numpy(S).cuda(), n)
    f = mvn().mvn_tlr_potrf(T, n, 1e-8)
    assert f.info == -1
    assert list(f.ranks.cpu().numpy()) == [r] * 6 and list(f.ranks_sigma.cpu().numpy()) == [r] * 6
    assert np.max(np.abs(dense_lower(T, n) - np.linalg.cholesky(S))) < 1e-11
    check_slots(f, T, n)


def test_tlr_potrf_eps_zero_is_dense(torch):
    """eps = 0 keeps every singular triplet: the factor is mvn_potrf's up to rounding."""
    cfg = W.small_config("tlrc0", 19, 100, 1, base="B")
    T, S, _ = sorted_cov(torch, cfg)
    n = cfg.n
    T2 = T.clone()
    f = mvn().mvn_tlr_potrf(T, n, 0.0)
    assert f.info == -1 and f.ranks.max().item() == 128
    assert mvn().mvn_potrf(T2, n) == -1
    assert np.max(np.abs(dense_lower(T, n) - dense_lower(T2, n))) < 1e-12


@pytest.mark.parametrize("base,g,eps,mode", [("B", 17, 1e-3, "abs"), ("B", 23, 1e-6, "abs"), ("C", 20, 1e-4, "abs"),
                                             ("B", 23, 1e-3, "fro"), ("A", 30, 1e-2, "abs")])
def test_tlr_potrf_vs_oracle(torch, base, g, eps, mode):
    cfg = W.small_config("tlrc", g, 100, 1, base=base)
    T, S, _ = sorted_cov(torch, cfg)
    n = cfg.n
    Tc = T.clone()
    rs_gpu_only = mvn().mvn_tlr_compress(Tc, n, eps, mode=1 if mode == "fro" else 0)
    Stg = dense_sym(Tc, n)
    mm = 1 if mode == "fro" else 0
    f = mvn().mvn_tlr_potrf(T, n, eps, mode=mm, raise_on_numeric=False)
    Lo, rLo, sLo, rSo, info_o = oracle.tlr_cholesky(S, eps, mode=mode)
    assert np.array_equal(f.ranks_sigma.cpu().numpy(), rs_gpu_only.cpu().numpy())
    assert (f.info == -1) == (info_o == -1)
    if f.info != -1:
        pytest.skip(f"TLR factorisation not SPD at eps={eps} (GPU row {f.info}, oracle row {info_o})")
    rL = f.ranks.cpu().numpy()
    diff = np.nonzero(rL != rLo)[0]
    for t in diff:
        lo, hi = sorted((int(rL[t]), int(rLo[t])))
        assert near_tie(sLo[t], eps, mode, lo, hi), (t, rL[t], rLo[t], sLo[t][lo - 1:hi + 1])
    G = dense_lower(T, n)
    if len(diff) == 0 and np.array_equal(f.ranks_sigma.cpu().numpy(), rSo):
        assert np.max(np.abs(G - Lo)) <= 1e-9, np.max(np.abs(G - Lo))
    check_slots(f, T, n)
    residual_identity(T, Stg, f, eps, n, mode)


def test_tlr_pipeline_vs_oracle(torch):
    """TLR Cholesky -> dense SOV -> log P_k: shared-L (the oracle's SOV on the GPU's L~) and
    independent (the oracle's TLR Cholesky and SOV) against the GPU."""
    import test_gpu_parity as P
    cfg = W.small_config("tlrcp", 23, 300, 2, base="B")
    T, S, a = sorted_cov(torch, cfg)
    n, eps = cfg.n, 1e-5
    f = mvn().mvn_tlr_potrf(T, n, eps)
    assert f.info == -1
    M, Sg = P.gpu_sov(torch, T, n, a, cfg.N, cfg.R, 5)
    lg = P.logp_from(M, Sg, cfg.NR)
    Lg = dense_lower(T, n)
    Mo, So = P.oracle_range(Lg, a, np.full(n, np.inf), cfg.N, cfg.R, 5, 0, cfg.NR)
    assert np.max(np.abs(lg - P.logp_from(Mo, So, cfg.NR))) <= 1e-10
    Lo, rLo, _, rSo, info_o = oracle.tlr_cholesky(S, eps)
    assert info_o == -1
    if np.array_equal(rLo, f.ranks.cpu().numpy()):
        Mi, Si = P.oracle_range(Lo, a, np.full(n, np.inf), cfg.N, cfg.R, 5, 0, cfg.NR)
        assert np.max(np.abs(lg - P.logp_from(Mi, Si, cfg.NR))) <= 1e-8


def test_tlr_potrf_failing_row_and_errors(torch):
    n = 300
    S = np.eye(n)
    S[200, 200] = -1.0
    T = mvn().mvn_pack_lower(torch.from_numpy(S).cuda(), n)
    f = mvn().mvn_tlr_potrf(T, n, 1e-3, raise_on_numeric=False)
    assert f.info == 200
    with pytest.raises(mvn().MvnError):
        mvn().mvn_tlr_potrf(mvn().mvn_pack_lower(torch.from_numpy(S).cuda(), n), n, 1e-3)
    # a rank above kmax is reported (MVN_E_NOMEM), not silently truncated
    rng = np.random.default_rng(5)
    F = rng.standard_normal((n, 20))
    S2 = F @ F.T + np.eye(n)
    with pytest.raises(mvn().MvnError) as ei:
        mvn().mvn_tlr_potrf(mvn().mvn_pack_lower(torch.from_numpy(S2).cuda(), n), n, 1e-10, kmax=8)
    assert ei.value.status == mvn().MVN_E_NOMEM
    f = mvn().mvn_tlr_potrf(mvn().mvn_pack_lower(torch.from_numpy(S2).cuda(), n), n, 1e-10, kmax=32)
    assert f.info == -1 and list(f.ranks.cpu().numpy()) == [20, 20, 20]
    Tb = mvn().alloc_tiles(n, "cuda")
    for eps, mode, kmax in [(-1.0, 0, 128), (1e-3, 2, 128), (1.5, 1, 128), (1e-3, 0, 0), (1e-3, 0, 129)]:
        with pytest.raises(mvn().MvnError):
            mvn().mvn_tlr_potrf(Tb, n, eps, mode=mode, kmax=kmax, U=torch.empty(1, dtype=torch.float64, device="cuda"),
                                V=torch.empty(1, dtype=torch.float64, device="cuda"))


def test_tlr_potrf_single_tile(torch):
    """n <= 128: no off-diagonal tile, the TLR factor is the dense one."""
    n = 100
    rng = np.random.default_rng(2)
    A = rng.standard_normal((n, n))
    S = A @ A.T / n + np.eye(n)
    T = mvn().mvn_pack_lower(torch.from_numpy(S).cuda(), n)
    f = mvn().mvn_tlr_potrf(T, n, 1e-3)
    assert f.info == -1
    assert np.max(np.abs(dense_lower(T, n) - np.linalg.cholesky(S))) < 1e-12


@pytest.mark.slow
@pytest.mark.parametrize("nu,beta,eps", [(1.5, 0.05, 1e-9), (0.5, 0.03, 1e-4)])
def test_tlr_potrf_sampled_large(torch, nu, beta, eps):
    """n = 16,384 (config C's grid; C's kernel nu = 3/2 at eps = 1e-9 — cond ~1e7, coarser eps loses
    positive definiteness — and D's nu = 1/2 kernel at 1e-4): the residual identity on sampled tiles
    of the GPU result, computed on the device from the factor's own rows."""
    cfg = W.small_config("tlrL", 128, 100, 1, base="C", nu=nu, beta=beta)
    import test_gpu_parity as P
    inp, order, a = P.sorted_inputs(cfg)
    xs = inp.xy[order]
    T = P.gpu_cov(torch, xs, cfg)
    n = cfg.n
    Tc = T.clone()
    mvn().mvn_tlr_compress(Tc, n, eps)
    f = mvn().mvn_tlr_potrf(T, n, eps)
    assert f.info == -1
    nt = -(-n // NB)
    rng = np.random.default_rng(0)
    tt = lambda X, I, J: X[((I * (I + 1)) // 2 + J) * NB * NB:((I * (I + 1)) // 2 + J + 1) * NB * NB].view(NB, NB).T
    for _ in range(12):
        I = int(rng.integers(1, nt))
        J = int(rng.integers(0, I + 1))
        acc = torch.zeros((NB, NB), dtype=torch.float64, device="cuda")
        for k in range(J + 1):
            acc += tt(T, I, k) @ tt(T, J, k).T
        R = (acc - tt(Tc, I, J)).cpu().numpy()
        nLJJ = np.linalg.norm(tt(T, J, J).cpu().numpy(), 2)
        if I == J:
            assert np.max(np.abs(np.tril(R))) < 1e-12 * nt
        else:
            assert np.linalg.norm(R, 2) < eps * nLJJ * (1 + 2e-6) + 1e-12 * nt, (I, J)
    assert 0 < f.ranks.max().item() <= 128


# ---- the factored SOV update (mvn_sov_prefix_tlr) ----

@pytest.mark.parametrize("base,g,eps,N,R,nb", [("B", 23, 1e-5, 300, 2, False), ("A", 30, 1e-3, 500, 1, True),
                                              ("B", 17, 1e-8, 250, 3, False)])
def test_sov_factored_update_vs_dense_and_oracle(torch, base, g, eps, N, R, nb):
    """The factored update reaches the dense sweep on the reconstructed L~ (summation order only) and
    the oracle's SOV on the same L~; ragged n, several sample blocks and shifts, a finite b."""
    import test_gpu_parity as P
    cfg = W.small_config("tlrsov", g, N, R, base=base)
    T, S, a = sorted_cov(torch, cfg)
    n = cfg.n
    f = mvn().mvn_tlr_potrf(T, n, eps)
    assert f.info == -1
    b = torch.from_numpy(a + 2.5).cuda() if nb else None
    bn = (a + 2.5) if nb else np.full(n, np.inf)
    Mt, St = mvn().mvn_sov_prefix_tlr(T, f, n, torch.from_numpy(a).cuda(), N, R, 5, b=b)
    Md, Sd = mvn().mvn_sov_prefix(T, n, torch.from_numpy(a).cuda(), N, R, 5, b=b)
    NR = N * R
    lt, ld = P.logp_from(Mt.cpu().numpy(), St.cpu().numpy(), NR), P.logp_from(Md.cpu().numpy(), Sd.cpu().numpy(), NR)
    assert np.max(np.abs(lt - ld)) <= 1e-11
    Mo, So = P.oracle_range(dense_lower(T, n), a, bn, N, R, 5, 0, NR)
    assert np.max(np.abs(lt - P.logp_from(Mo, So, NR))) <= 1e-10


def test_sov_factored_update_exact_low_rank_and_widths(torch):
    """Sigma = D + F F^T (exact rank 5 tiles): the factored sweep equals the oracle on numpy's
    Cholesky factor; sample ranges giving block widths 8 ... 128 (both GEMM fragment counts)."""
    import test_gpu_parity as P
    rng = np.random.default_rng(11)
    n, r = 400, 5
    F = rng.standard_normal((n, r)) * 0.3
    Sg = F @ F.T + np.diag(rng.uniform(0.5, 1.5, n))
    T = mvn().mvn_pack_lower(torch.from_numpy(Sg).cuda(), n)
    f = mvn().mvn_tlr_potrf(T, n, 1e-9)
    assert list(f.ranks.cpu().numpy()) == [r] * 6
    a = np.sort(rng.normal(-0.5, 0.5, n))
    da = torch.from_numpy(a).cuda()
    Lnp = np.linalg.cholesky(Sg)
    for begin, end in [(0, 148 * 8), (3, 3 + 148 * 40 + 17), (0, 148 * 128 + 300)]:
        Mt, St = mvn().mvn_sov_prefix_tlr(T, f, n, da, 10_000, 3, 9, begin, end)
        Mo, So = P.oracle_range(Lnp, a, np.full(n, np.inf), 10_000, 3, 9, begin, end)
        lt = P.logp_from(Mt.cpu().numpy(), St.cpu().numpy(), end - begin)
        assert np.max(np.abs(lt - P.logp_from(Mo, So, end - begin))) <= 1e-10


def test_sov_factored_update_errors(torch):
    n = 300
    T = mvn().alloc_tiles(n, "cuda")
    a = torch.zeros(n, dtype=torch.float64, device="cuda")
    f = mvn().TlrFactor(torch.zeros(1, dtype=torch.float64, device="cuda"), torch.zeros(1, dtype=torch.float64, device="cuda"),
                        torch.zeros(3, dtype=torch.int32, device="cuda"), torch.zeros(3, dtype=torch.int32, device="cuda"), 0, -1)
    with pytest.raises(mvn().MvnError):
        mvn().mvn_sov_prefix_tlr(T, f, n, a, 100, 1, 1)          # kmax = 0


def test_crd_tlr_end_to_end_vs_oracle(torch):
    """Alg. 1 end to end through the public mvn_crd with step (a) as the TLR Cholesky (MVN_CRD_TLR,
    P:319): against the oracle's pipeline on its own TLR factor (independent mode)."""
    cfg = W.small_config("crdtlr", 30, 2000, 4, base="A")
    inp = W.make_inputs(cfg)
    eps = 1e-6
    out = mvn().mvn_crd(inp.xy, inp.mu, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget, cfg.u, cfg.N, cfg.R,
                        cfg.seed_lattice, cfg.conf, method=mvn().CRD_TLR, tlr_eps=eps)
    var = np.full(cfg.n, cfg.sigma2 + cfg.nugget)
    order, a, _ = oracle.marginal_order(inp.mu, var, cfg.u)
    S = oracle.covariance(inp.xy[order], cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget)
    Lt, rL, sL, rS, info = oracle.tlr_cholesky(S, eps)
    assert out.info == -1 and info == -1
    ref = oracle.crd(inp.xy, inp.mu, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget, cfg.u, cfg.N, cfg.R,
                     cfg.seed_lattice, cfg.conf, chunk=500, nthreads=16, L=Lt)
    assert np.array_equal(out.order, ref.order)
    assert np.max(np.abs(out.logP - ref.logp)) <= 1e-8
    assert np.array_equal(out.k_star, ref.k_star) or np.any(ref.near_tie)
    dense = mvn().mvn_crd(inp.xy, inp.mu, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget, cfg.u, cfg.N, cfg.R,
                          cfg.seed_lattice, cfg.conf)
    assert np.max(np.abs(out.logP - dense.logP)) <= 1e-3          # eps = 1e-6 truncation
    with pytest.raises(mvn().MvnError):
        mvn().mvn_crd(inp.xy, inp.mu, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget, cfg.u, cfg.N, cfg.R,
                      cfg.seed_lattice, cfg.conf, method=mvn().CRD_TLR | mvn().CRD_POTRF_INT8, tlr_eps=eps)
