"""C-ABI argument validation on the GPU (errors are returned as MVN_E_USAGE, never thrown or
crashed; the Python binding raises MvnError): NaN / inverted limits, bad super-panel and column
filters, bad panel indices, bad MC method / range, posterior tiles without a matching posterior,
unsupported Matérn smoothness."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch(cuda_device):
    import torch as t
    return t


def mvn():
    import paper_2405_14892_b200 as m
    return m


def small_L(torch, n=200):
    xy = np.random.default_rng(0).uniform(size=(n, 2))
    T = mvn().mvn_cov_matern(torch.from_numpy(xy).cuda(), 1.0, 0.1, 0.5, 1e-8)
    assert mvn().mvn_potrf(T, n) == -1
    return T


def usage(fn, *a, **k):
    with pytest.raises(mvn().MvnError) as e:
        fn(*a, **k)
    assert e.value.status == mvn().MVN_E_USAGE, e.value


def test_sov_prefix_rejects_bad_limits(torch):
    n = 200
    T = small_L(torch, n)
    a = np.zeros(n)
    a[17] = math.nan
    usage(mvn().mvn_sov_prefix, T, n, torch.from_numpy(a).cuda(), 10, 1, 3)
    a = np.zeros(n)
    b = np.ones(n)
    b[5] = -1.0                                  # a_5 > b_5
    usage(mvn().mvn_sov_prefix, T, n, torch.from_numpy(a).cuda(), 10, 1, 3, b=torch.from_numpy(b).cuda())
    usage(mvn().mvn_sov_prefix, T, n, torch.zeros(n, dtype=torch.float64, device="cuda"), 10, 1, 3, 5, 5)   # empty range
    # a valid call afterwards still works (the context is not poisoned)
    M, S = mvn().mvn_sov_prefix(T, n, torch.zeros(n, dtype=torch.float64, device="cuda"), 10, 1, 3)
    assert torch.isfinite(M).all()


def test_potrf_building_blocks_reject_bad_arguments(torch):
    n = 5 * 128
    T = small_L(torch, n)
    usage(mvn().mvn_potrf_update, T, n, 2, 1, 2)          # col_first < k + kp
    usage(mvn().mvn_potrf_update, T, n, 0, 1, 1, 2, 3)    # col_block > col_stride
    usage(mvn().mvn_potrf_update, T, n, 0, 9, 10)         # kp > 8
    usage(mvn().mvn_potrf_panel, T, n, 5)                 # k >= nt
    buf = torch.empty(mvn().panel_numel(n, 0, 1), dtype=torch.float64, device="cuda")
    usage(mvn().mvn_panel_pack, T, n, 7, 1, buf)


def test_mc_and_posterior_and_matern_reject_bad_arguments(torch):
    n = 200
    T = small_L(torch, n)
    d_a = torch.zeros(n, dtype=torch.float64, device="cuda")
    usage(mvn().mvn_mc_validate, T, n, d_a, 1, 0, 100, method=3)
    usage(mvn().mvn_mc_validate, T, n, d_a, 1, 50, 50)
    xy = np.random.default_rng(1).uniform(size=(60, 2))
    mvn().mvn_posterior(xy, np.zeros(60), np.array([1, 5]), np.zeros(2), 1.0, 0.1, 0.5, 1e-8, 0.5)
    usage(mvn().mvn_posterior_tiles, np.arange(59))       # n differs from the last posterior
    usage(mvn().mvn_posterior_tiles, np.zeros(60, dtype=np.int64))   # not a permutation
    usage(mvn().mvn_cov_matern, torch.from_numpy(xy).cuda(), 1.0, 0.1, 0.0, 1e-8)   # nu must be in (0, 50]
    usage(mvn().mvn_cov_matern, torch.from_numpy(xy).cuda(), 1.0, 0.1, 51.0, 1e-8)
