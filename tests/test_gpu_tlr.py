"""NEXT-3 (part) on the GPU: fixed-accuracy TLR compression (mvn_tlr_compress, reading R23) against
the oracle (oracle/tlr.py: one LAPACK SVD per tile). Ranks must agree except where an oracle
singular value lies within 1e-12 of eps (a near tie, decided by rounding); the compressed tiles
agree to 1e-12 + 1e-13 sigma_1 (1 + sigma_1 / gap) (the Jacobi and gesdd subspaces of the same tile
differ by rounding / gap, gap = sigma_k - sigma_k+1); and the
GPU result satisfies Eckart-Young itself (||A - A_k||_2 = sigma_{k+1} < eps). The compressed matrix
then runs through POTRF + SOV and matches the oracle pipeline on the oracle's compressed matrix."""
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


def dense_sym(T, n):
    L = mvn().mvn_unpack_lower(T, n).T.contiguous().cpu().numpy()
    return np.tril(L) + np.tril(L, -1).T


def sorted_cov(torch, cfg):
    import test_gpu_parity as P
    inp, order, a = P.sorted_inputs(cfg)
    xs = inp.xy[order]
    T = P.gpu_cov(torch, xs, cfg)
    S = oracle.covariance(xs, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget)
    return T, S, a


def check_vs_oracle(T, S, ranks_gpu, eps, n, mode="abs"):
    St, ro, sig = oracle.tlr_compress(S, eps, mode=mode)
    G = dense_sym(T, n)
    nt = -(-n // NB)
    t = 0
    for I in range(1, nt):
        for J in range(I):
            k, ko = int(ranks_gpu[t]), int(ro[t])
            if k != ko:      # only a near tie at the threshold may differ
                lo, hi = min(k, ko), max(k, ko)
                if mode == "abs":
                    # the GPU drops the QR's trailing block once ||R_22||_F <= 1e-6 eps (kernels_tlr.cu),
                    # which moves a singular value by at most that
                    assert np.all(np.abs(sig[t][lo:hi] - eps) <= 1e-12 + 2e-6 * eps), (I, J, k, ko, sig[t][lo:hi])
                else:            # the smaller rank is feasible up to rounding of the tail sum
                    tot = np.sum(sig[t] ** 2)
                    assert np.sum(sig[t][lo:] ** 2) <= eps * eps * tot * (1 + 1e-9) + 1e-28, (I, J, k, ko)
            rs, cs = slice(I * NB, min((I + 1) * NB, n)), slice(J * NB, (J + 1) * NB)
            E = S[rs, cs] - G[rs, cs]
            if mode == "abs":
                e2 = np.linalg.norm(E, 2)
                assert (e2 < eps * (1 + 2e-6) + 1e-12) if eps > 0 else np.max(np.abs(E)) < 1e-13, (I, J, k, ko, e2, sig[t][max(k - 2, 0):k + 2])
            else:
                ef, af = np.linalg.norm(E), np.linalg.norm(S[rs, cs])
                assert ef <= eps * af * (1 + 1e-9) + 1e-13, (I, J, k, ko, ef, af)
            if k == ko:
                # the kept subspace of a tile moves by (rounding perturbation) / (sigma_k - sigma_k+1)
                sg = sig[t]
                gap = sg[k - 1] - sg[k] if 0 < k < NB else np.inf
                tau = 1e-6 * eps * (1.0 if mode == "abs" else np.linalg.norm(S[rs, cs]))   # the dropped R_22
                tol = 1e-12 + (1e-13 * sg[0] + tau) * (1.0 + sg[0] / gap)
                assert np.max(np.abs(G[rs, cs] - St[rs, cs])) <= tol, (I, J, k, gap)
            t += 1
    for I in range(nt):                       # diagonal tiles untouched
        rs = slice(I * NB, min((I + 1) * NB, n))
        assert np.array_equal(G[rs, rs], dense_sym(T, n)[rs, rs])
    return St, ro


@pytest.mark.parametrize("base,g", [("B", 23), ("C", 30), ("B", 17)])
@pytest.mark.parametrize("eps,mode", [(1e-1, "abs"), (1e-3, "abs"), (1e-6, "abs"), (1e-1, "fro"), (1e-4, "fro"),
                                      (1e-8, "fro")])
def test_tlr_compress_vs_oracle(torch, base, g, eps, mode):
    cfg = W.small_config(f"tlr{g}", g, 100, 1, base=base)
    T, S, _ = sorted_cov(torch, cfg)
    T0 = T.clone()
    n = cfg.n
    ranks = mvn().mvn_tlr_compress(T, n, eps, mode=0 if mode == "abs" else 1).cpu().numpy()
    nt = -(-n // NB)
    assert ranks.shape[0] == nt * (nt - 1) // 2 and ranks.min() >= 0 and ranks.max() <= NB
    check_vs_oracle(T, S, ranks, eps, n, mode)
    G0 = dense_sym(T0, n)
    G = dense_sym(T, n)
    for I in range(nt):
        rs = slice(I * NB, min((I + 1) * NB, n))
        assert np.array_equal(G[rs, rs], G0[rs, rs])


def test_tlr_exact_rank(torch):
    rng = np.random.default_rng(11)
    n = 300
    X = rng.standard_normal((n, 5))
    S = X @ X.T + np.diag(rng.uniform(1, 2, n))
    T = mvn().mvn_pack_lower(torch.from_numpy(S).cuda(), n)
    ranks = mvn().mvn_tlr_compress(T, n, 1e-9).cpu().numpy()
    assert list(ranks) == [5, 5, 5]
    assert np.max(np.abs(dense_sym(T, n) - S)) <= 1e-12 * np.max(np.abs(S))
    T = mvn().mvn_pack_lower(torch.from_numpy(S).cuda(), n)
    assert list(mvn().mvn_tlr_compress(T, n, 1e6).cpu().numpy()) == [0, 0, 0]
    G = dense_sym(T, n)
    assert not G[NB:2 * NB, :NB].any() and not G[2 * NB:, :2 * NB].any()


def test_tlr_eps_zero_full_rank(torch):
    rng = np.random.default_rng(12)
    n = 256
    A = rng.standard_normal((n, n))
    S = A @ A.T / n + np.eye(n)
    T = mvn().mvn_pack_lower(torch.from_numpy(S).cuda(), n)
    ranks = mvn().mvn_tlr_compress(T, n, 0.0).cpu().numpy()
    assert list(ranks) == [128]
    assert np.max(np.abs(dense_sym(T, n) - S)) <= 1e-13


def test_tlr_single_tile_is_noop(torch):
    n = 100
    rng = np.random.default_rng(13)
    xy = rng.uniform(size=(n, 2))
    T = mvn().mvn_cov_matern(torch.from_numpy(xy).cuda(), 1.0, 0.1, 0.5, 1e-8)
    T0 = T.clone()
    mvn().mvn_tlr_compress(T, n, 1e-2)
    assert torch.equal(T, T0)


def test_tlr_bad_args(torch):
    T = mvn().alloc_tiles(300, "cuda")
    for eps, mode in [(-1.0, 0), (1e-3, 2), (1.5, 1), (float("nan"), 0)]:
        with pytest.raises(mvn().MvnError):
            mvn().mvn_tlr_compress(T, 300, eps, mode=mode)


@pytest.mark.parametrize("eps", [1e-2, 1e-5])
def test_tlr_pipeline_vs_oracle(torch, eps):
    """Compressed Sigma -> POTRF -> SOV -> log P_k, against the oracle pipeline on its own compressed
    Sigma (shared sample range; the two compressed matrices differ at rounding level)."""
    import test_gpu_parity as P
    cfg = W.small_config("tlrp", 23, 300, 2, base="B")
    T, S, a = sorted_cov(torch, cfg)
    n = cfg.n
    ranks = mvn().mvn_tlr_compress(T, n, eps).cpu().numpy()
    St, ro = check_vs_oracle(T, S, ranks, eps, n)
    info = mvn().mvn_potrf(T, n, raise_on_numeric=False)
    Lo, info_o = oracle.cholesky(St)
    assert (info == -1) == (info_o < 0)
    if info != -1:
        pytest.skip("compressed Sigma not SPD at this eps")
    M, Sg = P.gpu_sov(torch, T, n, a, cfg.N, cfg.R, 5)
    Mo, So = P.oracle_range(Lo, a, np.full(n, np.inf), cfg.N, cfg.R, 5, 0, cfg.NR)
    lg, lo = P.logp_from(M, Sg, cfg.NR), P.logp_from(Mo, So, cfg.NR)
    assert np.max(np.abs(lg - lo)) <= 1e-9


def test_tlr_relative_mode_limits(torch):
    """Mode 1 (relative Frobenius) at its ends: eps = 1 drops every off-diagonal tile (k = 0 meets
    ||A - 0||_F <= ||A||_F), eps = 0 keeps every nonzero singular value (the tile is unchanged up to
    rounding); n a multiple of 128 (no ragged tile)."""
    rng = np.random.default_rng(21)
    n = 256
    A = rng.standard_normal((n, n))
    S = A @ A.T / n + np.eye(n)
    T = mvn().mvn_pack_lower(torch.from_numpy(S).cuda(), n)
    assert list(mvn().mvn_tlr_compress(T, n, 1.0, mode=1).cpu().numpy()) == [0]
    G = dense_sym(T, n)
    assert not G[128:, :128].any()
    assert np.array_equal(G[:128, :128], S[:128, :128]) and np.array_equal(G[128:, 128:], S[128:, 128:])
    T = mvn().mvn_pack_lower(torch.from_numpy(S).cuda(), n)
    assert list(mvn().mvn_tlr_compress(T, n, 0.0, mode=1).cpu().numpy()) == [128]
    assert np.max(np.abs(dense_sym(T, n) - S)) <= 1e-13


@pytest.mark.parametrize("eps", [1e-1, 1e-4])
def test_tlr_relative_mode_scale_invariant(torch, eps):
    """Mode 1 is a relative criterion, so compressing s * Sigma must give the same ranks and s times
    the same tiles for any scale s (here 2^-27: every tile norm far below eps, where an absolute
    Jacobi skip floor would leave the columns unrotated and break ||A - A_k||_F <= eps ||A||_F).
    Checked against the oracle on the scaled matrix with no absolute slack."""
    cfg = W.small_config("tlrs", 23, 100, 1, base="B")
    T, S, _ = sorted_cov(torch, cfg)
    n = cfg.n
    s = 2.0 ** -27                                # ~7.5e-9, exact scaling (power of two)
    Ts = T * s
    r1 = mvn().mvn_tlr_compress(T, n, eps, mode=1).cpu().numpy()
    rs = mvn().mvn_tlr_compress(Ts, n, eps, mode=1).cpu().numpy()
    _, ro, _ = oracle.tlr_compress(S * s, eps, mode="fro")
    assert np.array_equal(rs, r1)
    assert np.sum(rs != ro) <= 1                  # a near tie at most
    G, Gs = dense_sym(T, n), dense_sym(Ts, n)
    assert np.max(np.abs(Gs / s - G)) <= 1e-12 * np.max(np.abs(S))
    nt = -(-n // NB)
    for I in range(1, nt):
        for J in range(I):
            rsl, csl = slice(I * NB, min((I + 1) * NB, n)), slice(J * NB, (J + 1) * NB)
            ef = np.linalg.norm(S[rsl, csl] * s - Gs[rsl, csl])
            assert ef <= eps * np.linalg.norm(S[rsl, csl] * s) * (1 + 1e-9), (I, J)
