"""Edge sizes of the CUDA path vs the oracle (shared-L mode): n around the 64-row SOV block and the
128-row tile (1, 2, 63, 64, 65, 127, 128, 129), sample ranges of 1, 31, 33 and 200 draws
(narrow and ragged sample blocks, ranges across a shift boundary), and the MC validation at n = 1."""
import math

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch(cuda_device):
    import torch as t
    return t


def mvn():
    import paper_2405_14892_b200 as m
    return m


def logp(M, S, NR):
    with np.errstate(divide="ignore"):
        return np.where(S > 0, M + np.log(S) - math.log(NR), -np.inf)


@pytest.mark.parametrize("n", [1, 2, 63, 64, 65, 127, 128, 129])
@pytest.mark.parametrize("begin,end", [(0, 1), (7, 38), (50, 83), (90, 290)])
def test_sov_edge_sizes(torch, n, begin, end):
    import test_gpu_parity as P
    rng = np.random.default_rng(1000 + n)
    xy = rng.uniform(size=(n, 2))
    T = mvn().mvn_cov_matern(torch.from_numpy(xy).cuda(), 1.0, 0.15, 0.5, 1e-8)
    assert mvn().mvn_potrf(T, n) == -1
    a = np.sort(rng.uniform(-1.5, 0.5, n))
    N, R, seed = 100, 3, 17                           # ranges cross the shift boundaries at 100, 200
    M, S = P.gpu_sov(torch, T, n, a, N, R, seed, begin, end)
    L = P.to_dense_lower(T, n)
    Mo, So = P.oracle_range(L, a, np.full(n, np.inf), N, R, seed, begin, end, nthreads=4)
    assert np.max(np.abs(logp(M, S, end - begin) - logp(Mo, So, end - begin))) <= 1e-11


@pytest.mark.parametrize("method", [0, 1, 2])
def test_mc_single_site(torch, method):
    T = mvn().mvn_pack_lower(torch.from_numpy(np.array([[2.0]])).cuda(), 1)
    mvn().mvn_potrf(T, 1)
    N = 40_000
    cnt = mvn().mvn_mc_validate(T, 1, torch.tensor([0.5], dtype=torch.float64, device="cuda"), 5, 0, N,
                                method=method).cpu().numpy()
    from scipy.special import ndtr
    p = 1 - ndtr(0.5 / math.sqrt(2.0))
    assert abs(cnt[1] / N - p) <= 4 * math.sqrt(p * (1 - p) / N)
    f = oracle.mc_first(np.array([[math.sqrt(2.0)]]), np.array([0.5]), 5, 0, N)
    assert abs(int(cnt[1]) - int(np.sum(f >= 1))) <= 2      # same draws, rounding-level ties only


# ---------------------------------------------------------------------- b = +inf far tails (a8)
# The upper-exceedance fast path of k_sov forms each 8-row sub-block's log-sum-exp from a running
# product exp(ell - c_w) * prod q; it must fall back to the exact per-row path whenever that product
# underflows (reading R10), e.g. eight factors q ~ Phibar(14) ~ 8e-45 in a row.
@pytest.mark.parametrize("n", [16, 129])
@pytest.mark.parametrize("aval", [13.3, 13.5, 14.0, 20.0, 30.0, 34.9])
def test_sov_upper_far_tail_identity(torch, n, aval):
    """Sigma = I, b = NULL: log P_k = k log Phibar(a) exactly (zero variance); and = the oracle."""
    from scipy.special import log_ndtr
    import test_gpu_parity as P
    T = mvn().mvn_pack_lower(torch.from_numpy(np.eye(n)).cuda(), n)
    assert mvn().mvn_potrf(T, n) == -1
    a = np.full(n, aval)
    N, R = 96, 2
    M, S = P.gpu_sov(torch, T, n, a, N, R, 11)
    lp = logp(M, S, N * R)
    assert np.all(np.isfinite(lp))
    k = np.arange(1, n + 1)
    want = k * log_ndtr(-aval)
    assert np.all(np.abs(lp - want) <= 1e-12 + 4e-15 * np.abs(want)), np.max(np.abs(lp - want))
    Mo, So = P.oracle_range(np.eye(n), a, np.full(n, np.inf), N, R, 11, 0, N * R, nthreads=4)
    lo = logp(Mo, So, N * R)
    assert np.all(np.abs(lp - lo) <= 1e-12 + 4e-15 * np.abs(lo))


def test_sov_upper_far_tail_correlated(torch):
    """A correlated nu = 3/2 field (12 x 12 grid, beta = 0.02) with thresholds putting every
    conditional limit a' of every sample in the far tail [13, 35] (checked on the oracle's own
    y): GPU = oracle within 1e-12 relative, no -inf."""
    import test_gpu_parity as P
    g = 12
    n = g * g
    c = (np.arange(g) + 0.5) / g
    xy = np.stack(np.meshgrid(c, c, indexing="ij"), -1).reshape(-1, 2)
    T = mvn().mvn_cov_matern(torch.from_numpy(xy).cuda(), 1.0, 0.02, 1.5, 1e-8)
    assert mvn().mvn_potrf(T, n) == -1
    L = P.to_dense_lower(T, n)
    a = np.full(n, 22.0)
    N, R, seed = 64, 2, 23
    from oracle import lattice
    G, D = lattice.generators(n), lattice.shifts(seed, R, n)
    _, _, y = oracle.sov_unit(L, a, np.full(n, np.inf), G, D[0], 1, N, want_y=True)
    ap = (a[:, None] - (np.tril(L, -1) @ y)) / np.diag(L)[:, None]
    assert ap.min() >= 13.0 and ap.max() <= 35.0, (ap.min(), ap.max())
    M, S = P.gpu_sov(torch, T, n, a, N, R, seed)
    lp = logp(M, S, N * R)
    Mo, So = P.oracle_range(L, a, np.full(n, np.inf), N, R, seed, 0, N * R, nthreads=4)
    lo = logp(Mo, So, N * R)
    assert np.all(np.isfinite(lp))
    assert np.all(np.abs(lp - lo) <= 1e-12 + 1e-14 * np.abs(lo)), np.max(np.abs(lp - lo))


# ---------------------------------------------------------------------- sample-block widths
@pytest.mark.parametrize("per_cta", [9, 17, 45, 67, 70, 100, 121, 128, 300, 541])
def test_sov_block_widths(torch, per_cta):
    """Every sample-block width k_sov can pick (multiples of 8 up to 128; both GEMM warp layouts:
    2 x 4 for widths that are multiples of 32, 4 x 2 column halves otherwise, including the empty
    half at width 8) against the oracle in shared-L mode: 148 * per_cta samples give every
    persistent CTA per_cta samples (one block of 8 ceil(per_cta / 8), or several blocks of
    near-equal widths), across shift boundaries, n = 263 (five row blocks, a ragged tail)."""
    import test_gpu_parity as P
    n = 263
    rng = np.random.default_rng(77)
    xy = rng.uniform(size=(n, 2))
    T = mvn().mvn_cov_matern(torch.from_numpy(xy).cuda(), 1.0, 0.12, 1.5, 1e-8)
    assert mvn().mvn_potrf(T, n) == -1
    a = np.sort(rng.uniform(-2.0, 0.3, n))
    total = 148 * per_cta
    R = 3
    N = -(-total // R) + 5
    begin = 3
    end = begin + total
    M, S = P.gpu_sov(torch, T, n, a, N, R, 41, begin, end)
    L = P.to_dense_lower(T, n)
    Mo, So = P.oracle_range(L, a, np.full(n, np.inf), N, R, 41, begin, end, nthreads=8)
    d = np.max(np.abs(logp(M, S, total) - logp(Mo, So, total)))
    assert d <= 1e-11, d


# ---------------------------------------------------------------------- K6 block-slice boundaries
@pytest.mark.parametrize("count", [2, 15, 16, 17, 31, 33, 47])
def test_sov_reduce_slice_boundaries(torch, count):
    """K6 (`k_reduce_blocks`) combines the block partials in 16 contiguous slices: sample counts
    below the SM count give one sample block per sample, so `count` is the number of partials —
    fewer than, equal to and just above the slice count, with empty and ragged last slices — against
    the oracle in shared-L mode. The last limit (a = 60) puts every factor of the last prefix far below
    the fp64 range (log P_n ~ -4,000: the log-space path of reading R10), so the partials combined
    there differ by hundreds in their maxima."""
    import test_gpu_parity as P
    n = 70
    rng = np.random.default_rng(300 + count)
    xy = rng.uniform(size=(n, 2))
    T = mvn().mvn_cov_matern(torch.from_numpy(xy).cuda(), 1.0, 0.2, 0.5, 1e-8)
    assert mvn().mvn_potrf(T, n) == -1
    a = np.sort(rng.uniform(-1.5, 0.5, n))
    a[-1] = 60.0                                      # 1 - Phi(a') underflows fp64: log space only
    N, R, seed = 40, 2, 23
    begin, end = 11, 11 + count
    M, S = P.gpu_sov(torch, T, n, a, N, R, seed, begin, end)
    L = P.to_dense_lower(T, n)
    Mo, So = P.oracle_range(L, a, np.full(n, np.inf), N, R, seed, begin, end, nthreads=2)
    lg, lo = logp(M, S, count), logp(Mo, So, count)
    assert np.all(np.isfinite(lo)) and lo[-1] < -1000.0 and np.all(np.isfinite(lg))
    assert np.max(np.abs(lg[:-1] - lo[:-1])) <= 1e-11
    assert abs(lg[-1] - lo[-1]) <= 1e-12 * abs(lo[-1]), (lg[-1], lo[-1])
