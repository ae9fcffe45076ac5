"""NEXT-2 on the GPU: mvn_mc_validate (Monte-Carlo validation of the regions) against the
oracle (oracle/mcval.py) on the same seeded draws (reading R20).

Per-sample first failing rows f_s are integers decided by floating point: the GPU forms (L z)_k
with DMMA sums, the oracle with an ascending dot, and z comes from two independent Phi^{-1}
implementations (AS 241 vs Halley), so a decision x_k <= a_k may legitimately differ where
|x_k - a_k| is at rounding level. The bar: f_s identical for every sample whose oracle margin
min_k |x_k - a_k| / (1 + |a_k|) over the rows it examined exceeds 1e-9; the histogram equals the
bincount of the GPU's own f_s exactly; p_hat levels follow from the histogram exactly."""
import math

import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu
GAP = 1e-9


@pytest.fixture(scope="module")
def torch(cuda_device):
    import torch as t
    return t


def mvn():
    import paper_2405_14892_b200 as m
    return m


def dense(T, n):
    return mvn().mvn_unpack_lower(T, n).T.contiguous().cpu().numpy()


def factor(torch, cfg):
    inp = W.make_inputs(cfg)
    var = np.full(cfg.n, cfg.sigma2 + cfg.nugget)
    order, a, _ = oracle.marginal_order(inp.mu, var, cfg.u)
    T = mvn().mvn_cov_matern(torch.from_numpy(np.ascontiguousarray(inp.xy[order])).cuda(), cfg.sigma2, cfg.beta,
                             cfg.nu, cfg.nugget)
    assert mvn().mvn_potrf(T, cfg.n) == -1
    return T, a


def gpu_first(torch, T, n, a, seed, begin, end, method=0):
    d_a = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    first = torch.empty(end - begin, dtype=torch.int32, device="cuda")
    count = mvn().mvn_mc_validate(T, n, d_a, seed, begin, end, first=first, method=method)
    return first.cpu().numpy(), count.cpu().numpy().astype(np.int64)


def check_against_oracle(fg, L, a, seed, begin, end):
    fo, _, gap = oracle.mc_first(L, a, seed, begin, end - begin, nthreads=16, diagnostics=True)
    diff = fg != fo
    assert not np.any(diff & (gap > GAP)), np.flatnonzero(diff & (gap > GAP))[:10]
    return fo, int(diff.sum())


@pytest.mark.parametrize("method", [0, 1, 2])
@pytest.mark.parametrize("g,base,begin,end", [(20, "A", 0, 4096), (9, "A", 5, 700), (23, "C", 1000, 3333),
                                              (11, "A", 0, 129)])
def test_mc_first_vs_oracle(torch, g, base, begin, end, method):
    """method 0: X = L Z on fp64 DMMA; method 1: on the int8 tensor cores (tcgen05 Ozaki split)."""
    cfg = W.small_config(f"mc{g}", g, 100, 1, base=base)
    T, a = factor(torch, cfg)
    n = cfg.n
    fg, count = gpu_first(torch, T, n, a, 1234, begin, end, method)
    assert np.array_equal(count, np.bincount(fg, minlength=n + 1))
    fo, nd = check_against_oracle(fg, dense(T, n), a, 1234, begin, end)
    assert nd <= max(1, (end - begin) // 1000)


@pytest.mark.parametrize("method", [0, 1, 2])
def test_mc_multiple_row_tiles_and_far_rows(torch, method):
    """n = 961 (8 row tiles, ragged last) with limits pushed low so that draws survive deep into
    the sweep and the later row tiles decide."""
    cfg = W.small_config("mc-deep", 31, 100, 1, base="A")   # n = 961
    T, a = factor(torch, cfg)
    n = cfg.n
    a = a - 3.5
    fg, count = gpu_first(torch, T, n, a, 77, 0, 2000, method)
    assert fg.max() > 600                                   # the deep tiles were exercised
    check_against_oracle(fg, dense(T, n), a, 77, 0, 2000)


def test_mc_int8_emulation_matches_fp64_path(torch):
    """The two products decide identically except where |x_k - a_k| is at rounding level; at
    n = 4,900 (config B geometry, 39 row tiles incl. a ragged one) over 10,000 draws."""
    cfg = W.small_config("mc-oz", 70, 100, 1, base="B")
    T, a = factor(torch, cfg)
    n = cfg.n
    f0, c0 = gpu_first(torch, T, n, a, 9, 0, 10_000, 0)
    f1, c1 = gpu_first(torch, T, n, a, 9, 0, 10_000, 1)
    f2, c2 = gpu_first(torch, T, n, a, 9, 0, 10_000, 2)
    assert np.mean(f0 != f1) <= 1e-3 and np.mean(f0 != f2) <= 1e-3
    assert np.array_equal(c1, np.bincount(f1, minlength=n + 1))
    assert np.array_equal(f1, f2)            # same slices, same products: identical exact integer sums


@pytest.mark.parametrize("method", [0, 1, 2])
def test_mc_identity_closed_form_both_methods(torch, method):
    n, N = 300, 50_000
    T = mvn().mvn_pack_lower(torch.from_numpy(np.eye(n)).cuda(), n)
    a = np.full(n, -2.5)
    a[:3] = [-0.5, 0.0, -1.0]
    cnt = mvn().mvn_mc_validate(T, n, torch.from_numpy(a).cuda(), 3, 0, N, method=method).cpu().numpy()
    from scipy.special import ndtr
    ks = [1, 2, 3, 10, 100, 300]
    ph = mvn().mvn_mc_levels(cnt, N, ks)
    for k, p_hat in zip(ks, ph):
        p = float(np.prod(1 - ndtr(a[:k])))
        assert abs(p_hat - p) <= 4 * math.sqrt(p * (1 - p) / N) + 1e-12, (k, p_hat, p)


def test_mc_chunks_accumulate_and_split(torch):
    cfg = W.small_config("mc-split", 15, 100, 1, base="A")
    T, a = factor(torch, cfg)
    n = cfg.n
    d_a = torch.from_numpy(a).cuda()
    c1 = mvn().mvn_mc_validate(T, n, d_a, 5, 0, 3000)
    c2 = mvn().mvn_mc_validate(T, n, d_a, 5, 0, 1111)
    mvn().mvn_mc_validate(T, n, d_a, 5, 1111, 3000, count=c2)
    assert torch.equal(c1, c2)
    c3 = mvn().mvn_mc_validate(T, n, d_a, 5, 0, 3000)
    assert torch.equal(c1, c3)                                # deterministic


def test_mc_identity_closed_form(torch):
    n, N = 300, 100_000
    T = mvn().mvn_pack_lower(torch.from_numpy(np.eye(n)).cuda(), n)
    a = np.full(n, -2.5)
    a[:3] = [-0.5, 0.0, -1.0]
    cnt = mvn().mvn_mc_validate(T, n, torch.from_numpy(a).cuda(), 3, 0, N).cpu().numpy()
    from scipy.special import ndtr
    ks = [1, 2, 3, 10, 100, 300]
    ph = mvn().mvn_mc_levels(cnt, N, ks)
    for k, p_hat in zip(ks, ph):
        p = float(np.prod(1 - ndtr(a[:k])))
        assert abs(p_hat - p) <= 4 * math.sqrt(p * (1 - p) / N) + 1e-12, (k, p_hat, p)


def test_mc_levels_host():
    cnt = np.array([3, 0, 2, 5], dtype=np.uint64)
    assert list(mvn().mvn_mc_levels(cnt, 10, [0, 1, 2, 3])) == [1.0, 0.7, 0.7, 0.5]
    with pytest.raises(mvn().MvnError):
        mvn().mvn_mc_levels(cnt, 10, [4])


@pytest.mark.slow
@pytest.mark.parametrize("method", [0, 1, 2])
def test_mc_full_config_D_sampled(torch, method):
    """Config D (n = 65,536) at full size: 2,048 draws through the bench launch configuration; the
    oracle decides each draw from the leading 4,096 x 4,096 block of L (a draw whose first failure
    lies in the block is decided there; the GPU must then agree; draws that survive the block
    must also survive it on the GPU)."""
    import test_gpu_parity as P
    cfg = W.CONFIGS["D"]
    T, a = factor(torch, cfg)
    n, m = cfg.n, 4096
    fg, count = gpu_first(torch, T, n, a, 42, 10_000, 12_048, method)
    Lm = P.leading_block(T, n, m)
    fo, _, gap = oracle.mc_first(Lm, a[:m], 42, 10_000, 2048, nthreads=16, diagnostics=True)
    decided = fo < m
    assert decided.mean() > 0.9
    bad = decided & (fg != fo) & (gap > GAP)
    assert not np.any(bad)
    assert np.all(fg[~decided] >= m)


def test_mc_int8_cluster_variant():
    """The 2-CTA cluster variant of the int8 kernel (multicast of the shared L slices;
    MVN_MC_CLUSTER=2, read once per process, hence the subprocess) passes the same oracle tests."""
    import os
    import subprocess
    import sys
    if os.environ.get("MVN_MC_CLUSTER"):
        pytest.skip("already running under a fixed MVN_MC_CLUSTER")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu and not slow", "tests/test_gpu_mc.py",
                        "-k", "method and not cluster_variant"], cwd=root, env=dict(os.environ, MVN_MC_CLUSTER="2"),
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
