"""NEXT-1: the SOV sweep over row phases (mvn_sweep_begin / mvn_sweep_rows / mvn_sweep_end) and the
assembly of a phase's rows from distributed storage (mvn_drows_offset / mvn_drows_unpack), on one GPU.

The phased sweep runs the same kernels on the same samples in the same order as mvn_sov_prefix — a
phase boundary only stops and restarts the row loop, carrying each sample's log weight and Y history —
so (M, S) must be BITWISE equal to mvn_sov_prefix's, whose parity with the oracle is pinned in
test_gpu_parity. Each phase is given only its rows: everything else in the buffer it is handed is NaN.
The emulated distributed pipeline (virtual ranks with their own storage, as in test_gpu_potrf_dist)
factors Sigma on distributed storage and sweeps with every phase assembled from the ranks' pieces."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
NB = 128


@pytest.fixture(scope="module")
def torch(cuda_device):
    import torch as t
    return t


def mvn():
    import paper_2405_14892_b200 as m
    return m


def problem(torch, n, nu=1.5, seed=0):
    import workloads as W
    xy = np.random.default_rng(seed + n).uniform(size=(n, 2))
    beta = 0.1 if nu == 0.5 else 0.05
    d_xy = torch.from_numpy(xy).cuda()
    L = mvn().mvn_cov_matern(d_xy, 1.0, beta, nu, 1e-8)
    assert mvn().mvn_potrf(L, n) == -1
    a = torch.from_numpy(np.random.default_rng(seed + 1).normal(0.3, 1.0, n)).cuda()
    return d_xy, beta, L, a


def phased(torch, L, n, a, N, R, seed, begin, end, rows_per_phase, b=None, poison=True):
    nt = -(-n // NB)
    sw = mvn().mvn_sweep_begin(n, a, N, R, seed, begin, end, b=b)
    for tb in range(0, nt, rows_per_phase):
        te = min(tb + rows_per_phase, nt)
        if poison:                              # the phase's rows only; every other element NaN
            P = torch.full_like(L, float("nan"))
            lo, hi = mvn().tile_rows_range(tb, te)
            P[lo:hi] = L[lo:hi]
            rows = mvn().tile_rows_slice(P, tb, te)
        else:
            rows = mvn().tile_rows_slice(L, tb, te)
        mvn().mvn_sweep_rows(sw, rows, tb, te)
    return mvn().mvn_sweep_end(sw)


@pytest.mark.parametrize("n,N,R,begin,end,phase,with_b", [
    (700, 1500, 2, 0, 3000, 1, False),          # one tile row per phase
    (700, 1500, 2, 100, 2900, 2, True),         # finite b, a sample sub-range
    (1000, 20000, 2, 0, 40000, 3, False),       # 270 samples per CTA: 3 blocks each, ragged last phase
    (1000, 20000, 2, 0, 40000, 8, True),        # one phase = the whole sweep
    (129, 997, 3, 5, 2000, 1, False),           # n = 128 + 1: a one-row last tile
    (64, 500, 1, 0, 500, 1, False),             # one tile, one phase
])
def test_phased_sweep_bitwise_equals_one_sweep(torch, n, N, R, begin, end, phase, with_b):
    _, _, L, a = problem(torch, n)
    b = a + torch.from_numpy(np.random.default_rng(3).uniform(0.5, 3.0, n)).cuda() if with_b else None
    M0, S0 = mvn().mvn_sov_prefix(L, n, a, N, R, 11, begin, end, b=b)
    M1, S1 = phased(torch, L, n, a, N, R, 11, begin, end, phase, b=b)
    torch.cuda.synchronize()
    assert torch.equal(M1, M0) and torch.equal(S1, S0), \
        f"max |dM| {float((M1 - M0).abs().max())} max |dS| {float((S1 - S0).abs().max())}"
    assert bool(torch.isfinite(M1).all())


def test_sweep_call_order_is_checked(torch):
    n = 600
    _, _, L, a = problem(torch, n)
    sw = mvn().mvn_sweep_begin(n, a, 300, 1, 1)
    with pytest.raises(mvn().MvnError):
        mvn().mvn_sweep_rows(sw, mvn().tile_rows_slice(L, 1, 2), 1, 2)     # must start at row 0
    mvn().mvn_sweep_rows(sw, mvn().tile_rows_slice(L, 0, 2), 0, 2)
    with pytest.raises(mvn().MvnError):
        mvn().mvn_sweep_end(sw)                                          # rows 2.. missing
    with pytest.raises(mvn().MvnError):
        mvn().mvn_sweep_rows(sw, mvn().tile_rows_slice(L, 2, 9), 2, 9)     # past nt = 5
    mvn().mvn_sweep_rows(sw, mvn().tile_rows_slice(L, 2, 5), 2, 5)
    M, S = mvn().mvn_sweep_end(sw)
    M0, S0 = mvn().mvn_sov_prefix(L, n, a, 300, 1, 1)
    torch.cuda.synchronize()
    assert torch.equal(M, M0) and torch.equal(S, S0)
    sw2 = mvn().mvn_sweep_begin(n, a, 300, 1, 1)
    mvn().mvn_sweep_free(sw2)                                            # abandoned sweep
    with pytest.raises(mvn().MvnError):
        mvn().mvn_sweep_begin(n, a * float("nan"), 300, 1, 1)            # NaN limits


def locals_from(torch, d_xy, beta, n, W, P, nu=1.5):
    kp = mvn().mvn_potrf_panel_width(n)
    ds, locs = [], []
    for r in range(W):
        d = mvn().dtiles(n, W, r, kp, P)
        loc = mvn().alloc_dtiles(n, W, r, kp, prows=P)
        mvn().mvn_dcov_matern(d_xy, d, 1.0, beta, nu, 1e-8, loc)
        ds.append(d)
        locs.append(loc)
    return kp, ds, locs


@pytest.mark.parametrize("n,W,P", [(1000, 2, 1), (40 * NB + 77, 3, 1), (2000, 4, 2), (3000, 6, 3), (130, 3, 1)])
def test_drows_unpack_assembles_the_rows(torch, n, W, P):
    """Every phase's row slice, assembled from the W ranks' pieces (one contiguous range of each
    rank's storage), equals the same rows of the full buffer; the pieces partition the rows."""
    d_xy, beta, _, _ = problem(torch, n)
    full = mvn().mvn_cov_matern(d_xy, 1.0, beta, 1.5, 1e-8)
    kp, ds, locs = locals_from(torch, d_xy, beta, n, W, P)
    nt = -(-n // NB)
    for tb, te in [(0, 1), (0, nt), (1, min(4, nt)), (nt - 1, nt), (min(2, nt - 1), nt)]:
        lo, hi = mvn().tile_rows_range(tb, te)
        rows = torch.full((hi - lo,), float("nan"), dtype=torch.float64, device="cuda")
        total = 0
        for r in range(W):
            a, b = mvn().mvn_drows_offset(ds[r], tb), mvn().mvn_drows_offset(ds[r], te)
            total += b - a
            if b > a:
                mvn().mvn_drows_unpack(ds[r], locs[r][a:b], tb, te, rows)
        torch.cuda.synchronize()
        assert total == hi - lo
        assert torch.equal(rows, full[lo:hi]), (tb, te)
    assert mvn().mvn_drows_offset(ds[0], nt) * 8 == mvn().mvn_dtiles_bytes(n, W, 0, kp, P)
    assert mvn().mvn_drows_offset(ds[0], nt + 1) == -1


@pytest.mark.parametrize("n,W,P,phase", [(1000, 2, 1, 2), (40 * NB + 77, 3, 1, 8), (2000, 4, 2, 3), (3000, 6, 3, 5)])
def test_emulated_distributed_pipeline(torch, n, W, P, phase):
    """NEXT-1 end to end on virtual ranks: Sigma generated on distributed storage, the distributed
    Cholesky (1-D or 2-D), then each rank's sample shard swept phase by phase with every phase's
    rows assembled from all ranks' pieces (the NCCL broadcasts are device copies here). Every rank's
    (M, S) is bitwise that of mvn_sov_prefix on the single-GPU factor for the same shard."""
    from test_gpu_potrf_dist import emulate, emulate_2d
    from paper_2405_14892_b200.parallel import shard_range, sov_phases
    d_xy, beta, L, a = problem(torch, n)
    kp, ds, locs = locals_from(torch, d_xy, beta, n, W, P)
    info = emulate(torch, locs, n, local=True) if P == 1 else emulate_2d(torch, locs, n, P, W // P)
    assert info == -1
    N, R = 4000, 2
    nt = -(-n // NB)
    phases = sov_phases(nt, phase)
    sws = []
    for g in range(W):
        b, e = shard_range(N * R, g, W)
        sws.append((b, e, mvn().mvn_sweep_begin(n, a, N, R, 5, b, e)))
    for tb, te in phases:
        lo, hi = mvn().tile_rows_range(tb, te)
        for g in range(W):                      # each rank assembles the phase from every piece
            rows = torch.full((hi - lo,), float("nan"), dtype=torch.float64, device="cuda")
            for r in range(W):
                x, y = mvn().mvn_drows_offset(ds[r], tb), mvn().mvn_drows_offset(ds[r], te)
                if y > x:
                    piece = locs[r][x:y].clone()                # the received copy
                    mvn().mvn_drows_unpack(ds[r], piece, tb, te, rows)
            mvn().mvn_sweep_rows(sws[g][2], rows, tb, te)
    for b, e, sw in sws:
        M, S = mvn().mvn_sweep_end(sw)
        M0, S0 = mvn().mvn_sov_prefix(L, n, a, N, R, 5, b, e)
        torch.cuda.synchronize()
        assert torch.equal(M, M0) and torch.equal(S, S0), (b, e)


def test_sov_distributed_single_rank(torch):
    """parallel.sov_distributed without a process group (one rank, no collectives) on 1-D storage
    holding all tiles."""
    from paper_2405_14892_b200.parallel import sov_distributed
    n = 1500
    d_xy, beta, L, a = problem(torch, n)
    kp, ds, locs = locals_from(torch, d_xy, beta, n, 1, 1)
    from test_gpu_potrf_dist import emulate
    assert emulate(torch, locs, n, local=True) == -1
    M, S = sov_distributed(locs[0], n, a, 3000, 2, 9, 0, 6000, kp, phase_rows=4)
    M0, S0 = mvn().mvn_sov_prefix(L, n, a, 3000, 2, 9)
    torch.cuda.synchronize()
    assert torch.equal(M, M0) and torch.equal(S, S0)
