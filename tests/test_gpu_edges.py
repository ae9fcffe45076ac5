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
