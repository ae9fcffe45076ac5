"""Multi-rank host logic of the multi-GPU path on CPU (gloo, world_size 2): sample sharding and the
per-prefix log-sum-exp combine (all_reduce MAX, rescale, all_reduce SUM) reproduce the
single-process estimate. Per-rank partials come from the oracle (no GPU needed)."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2405_14892_b200.parallel import combine_prefix, shard_range


def test_shard_range_covers_and_balances():
    for total in (2, 7, 100, 80_000, 400_000, 100_001):
        for world in (1, 2, 3, 4, 8):
            if total < world:
                continue
            rs = [shard_range(total, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == total
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            sizes = [e - b for b, e in rs]
            assert max(sizes) - min(sizes) <= 1
    assert shard_range(80_000, 3, 8) == (30_000, 40_000)     # config D at 8 GPUs: one shift per rank
    with pytest.raises(ValueError):
        shard_range(1, 0, 2)


def torch_rescale(Mg, M, S):
    """CPU stand-in for the CUDA kernel behind mvn_prefix_rescale (same definition, include/mvn.h)."""
    f = torch.where(M == -math.inf, torch.zeros_like(S), torch.exp(M - Mg))
    S.mul_(f)
    M.copy_(Mg)


def problem():
    import oracle
    rng = np.random.default_rng(11)
    n, N, R, seed = 40, 300, 3, 5
    S = oracle.covariance(rng.uniform(size=(n, 2)), 1.0, 0.15, 1.5, 1e-8)
    L, _ = oracle.cholesky(S)
    a = np.sort(rng.uniform(-1.2, 0.4, n))
    return L, a, N, R, seed


def range_partial(L, a, N, R, seed, begin, end):
    import oracle
    from oracle import lattice
    n = L.shape[0]
    G, D = lattice.generators(n), lattice.shifts(seed, R, n)
    parts, g = [], begin
    while g < end:
        r, j0 = g // N, g % N + 1
        J = min(end - g, N - j0 + 1)
        parts.append(oracle.sov_unit(L, a, np.full(n, np.inf), G, D[r], j0, J)[0])
        g += J
    return oracle.combine_units(np.array(parts))


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    L, a, N, R, seed = problem()
    b, e = shard_range(N * R, rank, world)
    M, S = range_partial(L, a, N, R, seed, b, e)
    Mt, St = torch.from_numpy(M.copy()), torch.from_numpy(S.copy())
    combine_prefix(Mt, St, rescale=torch_rescale)
    out[rank] = (Mt.numpy().copy(), St.numpy().copy())
    dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_combine_matches_single_process(world):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, free_port(), out), nprocs=world, join=True)
    L, a, N, R, seed = problem()
    M1, S1 = range_partial(L, a, N, R, seed, 0, N * R)
    lp1 = M1 + np.log(S1) - math.log(N * R)
    for r in range(world):
        M, S = out[r]
        lp = M + np.log(S) - math.log(N * R)
        assert np.max(np.abs(lp - lp1)) <= 1e-13
    assert np.array_equal(out[0][0], out[world - 1][0])        # every rank holds the same result


# ------------------------------------------------------------------ deterministic per-unit combine
def units_partial(L, a, N, R, seed, u0, u1):
    """Oracle per-unit partials [u1-u0][n][2] for 128-sample units of the global sample index."""
    import oracle
    from oracle import lattice
    n = L.shape[0]
    G, D = lattice.generators(n), lattice.shifts(seed, R, n)
    out = []
    for u in range(u0, u1):
        g, ge = 128 * u, min(128 * u + 128, N * R)
        parts = []
        while g < ge:                              # a unit can straddle a shift boundary
            r, j0 = g // N, g % N + 1
            J = min(ge - g, N - j0 + 1)
            parts.append(oracle.sov_unit(L, a, np.full(n, np.inf), G, D[r], j0, J)[0])
            g += J
        M, S = oracle.combine_units(np.array(parts))
        out.append(np.stack([M, S], -1))
    return np.array(out)


def host_reduce(P):
    import oracle
    M, S = oracle.combine_units(P.numpy())
    return torch.from_numpy(M), torch.from_numpy(S)


def _worker_units(rank, world, port, out):
    from paper_2405_14892_b200.parallel import combine_units_deterministic
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    L, a, N, R, seed = problem()
    U = -(-N * R // 128)
    u0, u1 = shard_range(U, rank, world)
    P = torch.from_numpy(units_partial(L, a, N, R, seed, u0, u1))
    M, S = combine_units_deterministic(P, reduce=host_reduce)
    out[rank] = (M.numpy().copy(), S.numpy().copy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_deterministic_unit_combine_is_bitwise_W_independent(world):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_units, args=(world, free_port(), out), nprocs=world, join=True)
    L, a, N, R, seed = problem()
    U = -(-N * R // 128)
    M1, S1 = host_reduce(torch.from_numpy(units_partial(L, a, N, R, seed, 0, U)))
    for r in range(world):
        M, S = out[r]
        assert np.array_equal(M, M1.numpy()) and np.array_equal(S, S1.numpy())
