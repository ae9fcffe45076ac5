"""ORACLE (test infrastructure only) — NEXT-3 (part), Tile Low-Rank compression at a fixed accuracy.

PAPER.md §II-C: TLR "is based on the separate approximation of each tile using the
Singular Value Decomposition (SVD) ... the ranks of the tiles correspond to the most significant
singular values"; Alg. 1 l.7: pmvn_init "encompasses the compression of the covariance
matrix Sigma into the TLR format". Reading R23: the matrix is cut into nb x nb tiles
(nb = 128, the last tile zero-padded); the diagonal tiles stay dense; every off-diagonal tile A keeps
its k largest singular triplets and is replaced by U_k S_k V_k^T, k from the accuracy eps:
mode "abs": k = #{sigma_i >= eps}; mode "fro": the smallest k with ||A - A_k||_F <= eps ||A||_F
(relative per tile; the paper does not state its convention, both are offered).
One library SVD (numpy.linalg.svd, LAPACK gesdd) per tile, fp64. Pinned in tests/test_oracle_tlr.py
against Eckart-Young (spectral error = sigma_{k+1} < eps, Frobenius error^2 = sum of the dropped
sigma_i^2), exact-rank tiles, eps = 0 (identity), and singular values from an independent route
(eigenvalues of A^T A).
"""
from __future__ import annotations

import numpy as np

NB = 128


def tile_svd(A: np.ndarray):
    """Singular values (descending) and factors of one tile."""
    U, s, Vt = np.linalg.svd(A)
    return U, s, Vt


def rank_for(s: np.ndarray, eps: float, mode: str = "abs") -> int:
    """k from the singular values s (descending) and the accuracy eps (R23)."""
    if mode == "abs":
        return int(np.count_nonzero((s >= eps) & (s > 0.0)))
    tot = float(np.sum(s ** 2))
    k = len(s)
    tail = 0.0
    while k > 0 and tail + s[k - 1] ** 2 <= eps * eps * tot:   # drop the smallest while within budget
        tail += s[k - 1] ** 2
        k -= 1
    return k


def compress_tile(A: np.ndarray, eps: float, mode: str = "abs"):
    """(A_tilde, k, s): rank-k truncation (R23)."""
    U, s, Vt = tile_svd(A)
    k = rank_for(s, eps, mode)
    return (U[:, :k] * s[:k]) @ Vt[:k, :], k, s


def tlr_compress(S: np.ndarray, eps: float, nb: int = NB, mode: str = "abs"):
    """Symmetric S (n x n) -> (S_tilde, ranks, sigmas). ranks[I(I-1)/2 + J] for tile (I, J), I > J;
    S_tilde is symmetric, diagonal tiles equal to S's."""
    S = np.asarray(S, dtype=np.float64)
    n = S.shape[0]
    nt = -(-n // nb)
    P = np.zeros((nt * nb, nt * nb))
    P[:n, :n] = S
    out = P.copy()
    ranks = np.zeros(max(nt * (nt - 1) // 2, 0), dtype=np.int64)
    sig = np.zeros((len(ranks), nb))
    for I in range(1, nt):
        for J in range(I):
            A = P[I * nb:(I + 1) * nb, J * nb:(J + 1) * nb]
            At, k, s = compress_tile(A, eps, mode)
            t = I * (I - 1) // 2 + J
            ranks[t], sig[t] = k, s
            out[I * nb:(I + 1) * nb, J * nb:(J + 1) * nb] = At
            out[J * nb:(J + 1) * nb, I * nb:(I + 1) * nb] = At.T
    return out[:n, :n], ranks, sig


def tlr_cholesky(S: np.ndarray, eps: float, nb: int = NB, mode: str = "abs"):
    """NEXT-3: the TLR Cholesky of Alg. 1 l.7-8 ("compression of the covariance matrix into the
    TLR format", box (a) "can be performed using both dense and TLR computations"), reading
    R26: Sigma is compressed at eps (tlr_compress, R23), then the tile columns are
    factored left to right; for column j

        T_i  = Stilde_ij - sum_{k<j} Ltilde_ik Ltilde_jk^T      (i >= j; every Ltilde_ik low rank)
        L_jj = chol(T_j)                                       (dense diagonal tile)
        L_ij = T_i L_jj^{-T}                                   (i > j)
        Ltilde_ij = rank-k truncation of L_ij at eps            (R23's rule, one SVD per tile)

    i.e. every off-diagonal tile of L is truncated once, when its column is complete (the updates
    are applied to the exact low-rank products, not re-truncated after each one; reading R26).
    Library primitives per step: the oracle's Crout Cholesky (C) for L_jj, a triangular solve for
    L_ij, numpy's SVD for the truncation.

    Returns (Ltilde, ranks_L, sig_L, ranks_S, info): Ltilde n x n lower (low-rank tiles
    reconstructed), ranks_L / ranks_S the ranks of L's / Sigma's off-diagonal tiles at
    I(I-1)/2 + J, sig_L the singular values of each L_ij before truncation (near-tie detection),
    info = -1 or the first failing global row (then Ltilde is partial)."""
    import scipy.linalg as sla
    from .pipeline import cholesky as crout

    S = np.asarray(S, dtype=np.float64)
    n = S.shape[0]
    nt = -(-n // nb)
    St, ranks_S, _ = tlr_compress(S, eps, nb, mode)
    L = np.zeros((n, n))
    ranks_L = np.zeros(max(nt * (nt - 1) // 2, 0), dtype=np.int64)
    sig_L = np.zeros((len(ranks_L), nb))

    def blk(I):
        return slice(I * nb, min((I + 1) * nb, n))

    for j in range(nt):
        cj = blk(j)
        T = St[j * nb:, cj] - L[j * nb:, :j * nb] @ L[cj, :j * nb].T      # sum over k < j, tile by tile equal
        Ljj, info = crout(T[:cj.stop - cj.start])
        if info >= 0:
            return L, ranks_L, sig_L, ranks_S, j * nb + info
        L[cj, cj] = Ljj
        for I in range(j + 1, nt):
            rI = blk(I)
            Tij = T[rI.start - j * nb:rI.stop - j * nb]
            Lij = sla.solve_triangular(Ljj, Tij.T, lower=True).T            # T_i L_jj^{-T}
            P = np.zeros((nb, nb))
            P[:Lij.shape[0], :Lij.shape[1]] = Lij
            Lt, k, s = compress_tile(P, eps, mode)
            t = I * (I - 1) // 2 + j
            ranks_L[t], sig_L[t] = k, s
            L[rI, cj] = Lt[:Lij.shape[0], :Lij.shape[1]]
    return L, ranks_L, sig_L, ranks_S, -1
