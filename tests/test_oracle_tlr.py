"""Pins for oracle/tlr.py (NEXT-3 part, reading R23) against what the mathematics fixes:
Eckart-Young optimality of the truncated SVD, exact-rank tiles, eps = 0, and singular values
computed by an independent route (eigenvalues of A^T A, LAPACK syevd instead of gesdd)."""
import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.filterwarnings("ignore")


def test_exact_rank_tiles():
    rng = np.random.default_rng(3)
    n, nb = 300, 128                            # 3 tile rows, ragged last tile
    X = rng.standard_normal((n, 5))
    S = X @ X.T + np.diag(rng.uniform(1, 2, n))  # off-diagonal blocks have rank <= 5
    St, ranks, _ = oracle.tlr_compress(S, 1e-10)
    assert list(ranks) == [5, 5, 5]
    assert np.max(np.abs(St - S)) < 1e-12
    St0, r0, _ = oracle.tlr_compress(S, 1e3)   # above every singular value: off-diagonal tiles vanish
    assert list(r0) == [0, 0, 0]
    for I in range(3):
        sl = slice(I * nb, min((I + 1) * nb, n))
        assert np.array_equal(St0[sl, sl], S[sl, sl])
    St0[:nb, :nb] = 0; St0[nb:2 * nb, nb:2 * nb] = 0; St0[2 * nb:, 2 * nb:] = 0
    assert not St0.any()


def test_eps_zero_is_identity():
    rng = np.random.default_rng(4)
    A = rng.standard_normal((260, 260))
    S = A @ A.T
    St, ranks, _ = oracle.tlr_compress(S, 0.0)
    assert ranks[0] == 128
    assert np.max(np.abs(St - S)) < 1e-10 * np.max(np.abs(S))


@pytest.mark.parametrize("eps", [1e-1, 1e-3, 1e-6])
def test_eckart_young(eps):
    cfg = W.small_config("tlr", 16, 10, 1, base="B")
    inp = W.make_inputs(cfg)
    S = oracle.covariance(inp.xy, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget)
    St, ranks, sig = oracle.tlr_compress(S, eps)
    nb, t = 128, 0
    for I in range(1, 2):
        for J in range(I):
            A = S[I * nb:(I + 1) * nb, J * nb:(J + 1) * nb]
            E = A - St[I * nb:(I + 1) * nb, J * nb:(J + 1) * nb]
            k = ranks[t]
            # independent singular values: eig(A^T A) = sigma^2, each within eps_mach * sigma_1^2
            ev = np.linalg.eigvalsh(A.T @ A)[::-1]
            assert np.allclose(ev, sig[t] ** 2, rtol=1e-10, atol=1e-13 * sig[t][0] ** 2)
            s2 = np.linalg.norm(E, 2)
            tail = sig[t][k] if k < nb else 0.0
            assert abs(s2 - tail) <= 1e-12 + 1e-10 * tail and s2 < eps
            assert abs(np.linalg.norm(E) ** 2 - np.sum(sig[t][k:] ** 2)) <= 1e-12 * max(1.0, np.sum(sig[t] ** 2))
            assert k == 0 or sig[t][k - 1] >= eps
            t += 1
    assert np.allclose(St, St.T, atol=0, rtol=0)


def test_rank_monotone_in_eps():
    cfg = W.small_config("tlr", 20, 10, 1, base="B")
    inp = W.make_inputs(cfg)
    S = oracle.covariance(inp.xy, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget)
    prev = None
    for eps in [1e-1, 1e-2, 1e-4, 1e-8]:
        _, r, _ = oracle.tlr_compress(S, eps)
        if prev is not None:
            assert np.all(r >= prev)
        prev = r
    assert prev.max() <= 128


@pytest.mark.parametrize("eps", [0.3, 1e-2, 1e-4])
def test_relative_frobenius_mode(eps):
    """mode "fro": ||A - A_k||_F <= eps ||A||_F, and k is minimal (rank k - 1 violates it) —
    Eckart-Young in the Frobenius norm, with the error from the matrix itself, not from s."""
    cfg = W.small_config("tlr", 16, 10, 1, base="B")
    inp = W.make_inputs(cfg)
    S = oracle.covariance(inp.xy, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget)
    St, ranks, sig = oracle.tlr_compress(S, eps, mode="fro")
    A = S[128:256, :128]
    E = A - St[128:256, :128]
    k = int(ranks[0])
    assert np.linalg.norm(E) <= eps * np.linalg.norm(A) * (1 + 1e-12)
    if k > 0:
        U, s, Vt = np.linalg.svd(A)
        Ak1 = (U[:, :k - 1] * s[:k - 1]) @ Vt[:k - 1]
        assert np.linalg.norm(A - Ak1) > eps * np.linalg.norm(A)
    _, r_abs, _ = oracle.tlr_compress(S, eps * np.linalg.norm(A), mode="abs")
    assert 0 <= k <= 128 and r_abs[0] >= 0


# ---- NEXT-3: the TLR Cholesky (oracle/tlr.py tlr_cholesky, reading R26) ----

def _matern(g, base="B", nu=None):
    cfg = W.small_config("tlr", g, 10, 1, base=base)
    inp = W.make_inputs(cfg)
    return oracle.covariance(inp.xy, cfg.sigma2, cfg.beta, cfg.nu if nu is None else nu, cfg.nugget)


def test_tlr_cholesky_eps_zero_is_dense_cholesky():
    """eps = 0 keeps every singular triplet: the factor is the dense Crout factor (rounding only)."""
    S = _matern(19)                                       # n = 361: 3 tile rows, ragged last tile
    L, rL, _, rS, info = oracle.tlr_cholesky(S, 0.0)
    Ld, infod = oracle.cholesky(S)
    assert info == -1 and infod == -1
    assert np.all(rS == 128) and rL.max() == 128 and len(rL) == 3
    assert np.max(np.abs(L - Ld)) < 1e-12


def test_tlr_cholesky_diag_plus_low_rank_is_exact():
    """Sigma = D + F F^T (F of rank r): every off-diagonal tile of Sigma AND of its Cholesky factor
    has rank exactly r (the factor of a diagonal-plus-rank-r matrix is semiseparable of rank r), so
    with eps far below the kept and far above the dropped singular values the TLR factor is the exact
    Cholesky factor."""
    rng = np.random.default_rng(7)
    n, r = 450, 6
    F = rng.standard_normal((n, r))
    S = F @ F.T + np.diag(rng.uniform(1.0, 3.0, n))
    L, rL, sL, rS, info = oracle.tlr_cholesky(S, 1e-8)
    assert info == -1
    assert list(rS) == [r] * 6 and list(rL) == [r] * 6
    assert np.max(np.abs(L - np.linalg.cholesky(S))) < 1e-12
    assert np.all(sL[:, r] < 1e-12) and np.all(sL[:, r - 1] > 1e-6)


@pytest.mark.parametrize("eps,mode", [(1e-2, "abs"), (1e-4, "abs"), (1e-6, "abs"), (1e-3, "fro")])
def test_tlr_cholesky_residual_is_the_truncation(eps, mode):
    """What the algorithm fixes: (Ltilde Ltilde^T - Stilde)_IJ = (L_IJ - Ltilde_IJ) L_JJ^T for I > J
    and 0 on the diagonal tiles (T_J = L_JJ L_JJ^T), so the off-diagonal residual is bounded by the
    dropped singular value times ||L_JJ||_2 — a dropped update term, a transposed operand or a wrong
    tile index breaks it."""
    S = _matern(20, base="C", nu=1.5) if mode == "abs" and eps < 1e-5 else _matern(20)
    nb = 128
    L, rL, sL, rS, info = oracle.tlr_cholesky(S, eps, mode=mode)
    assert info == -1
    St, rS2, _ = oracle.tlr_compress(S, eps, mode=mode)
    assert np.array_equal(rS, rS2)
    R = L @ L.T - St
    n, nt = S.shape[0], -(-S.shape[0] // nb)
    scale = np.max(np.abs(S))
    for J in range(nt):
        cJ = slice(J * nb, min((J + 1) * nb, n))
        assert np.max(np.abs(R[cJ, cJ])) < 1e-13 * scale * nt
        nLJJ = np.linalg.norm(L[cJ, cJ], 2)
        for I in range(J + 1, nt):
            rI = slice(I * nb, min((I + 1) * nb, n))
            t = I * (I - 1) // 2 + J
            k = rL[t]
            tail = sL[t][k] if k < nb else 0.0
            res = np.linalg.norm(R[rI, cJ], 2)
            assert res <= tail * nLJJ * (1 + 1e-8) + 1e-13 * scale * nt
            if mode == "abs":
                assert res < eps * nLJJ
                assert k == 0 or sL[t][k - 1] >= eps
    assert rL.max() <= 128 and rL.min() >= 0


def test_tlr_cholesky_reports_the_failing_row():
    """A non-positive pivot at a known row (off-diagonal tiles zero: rank 0) is reported there."""
    n = 300
    S = np.eye(n)
    S[200, 200] = -1.0
    L, rL, _, rS, info = oracle.tlr_cholesky(S, 1e-3)
    assert info == 200
    assert np.all(rS == 0)
    S[200, 200] = 1.0
    L, rL, _, _, info = oracle.tlr_cholesky(S, 1e-3)
    assert info == -1 and np.array_equal(L, np.eye(n)) and np.all(rL == 0)
