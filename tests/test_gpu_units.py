"""Per-unit partials of the SOV sweep (mvn_sov_prefix_units / mvn_prefix_reduce) and
the bitwise-deterministic multi-GPU combine of §8(e): a unit's partial does not depend on how the
units are split over calls, so splitting the units over W "ranks" and reducing the concatenation in
unit order reproduces the single call bit for bit; against the oracle's per-unit partials on the
same L (shared-L mode) and against the sample-mode sweep within rounding."""
import math

import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch(cuda_device):
    import torch as t
    return t


def mvn():
    import paper_2405_14892_b200 as m
    return m


def setup(torch, g=21, N=700, R=3, base="C"):
    import test_gpu_parity as P
    cfg = W.small_config(f"u{g}", g, N, R, base=base)
    inp, order, a = P.sorted_inputs(cfg)
    T = P.gpu_cov(torch, inp.xy[order], cfg)
    assert mvn().mvn_potrf(T, cfg.n) == -1
    return cfg, T, a


@pytest.mark.parametrize("splits", [[0, 17], [0, 5, 11, 17], [0, 1, 2, 16, 17]])
def test_units_split_is_bitwise(torch, splits):
    cfg, T, a = setup(torch)
    n = cfg.n
    U = mvn().sov_units(cfg.N, cfg.R)
    assert U == 17
    d_a = torch.from_numpy(a).cuda()
    whole = mvn().mvn_sov_prefix_units(T, n, d_a, cfg.N, cfg.R, cfg.seed_lattice, 0, U)
    parts = [mvn().mvn_sov_prefix_units(T, n, d_a, cfg.N, cfg.R, cfg.seed_lattice, u0, u1)
             for u0, u1 in zip(splits[:-1], splits[1:])]
    assert torch.equal(torch.cat(parts, 0), whole)
    M, S = mvn().mvn_prefix_reduce(whole)
    M2, S2 = mvn().mvn_prefix_reduce(torch.cat(parts, 0))
    assert torch.equal(M, M2) and torch.equal(S, S2)
    # the sample-mode sweep (another block partition): equal up to summation order
    Ms, Ss = mvn().mvn_sov_prefix(T, n, d_a, cfg.N, cfg.R, cfg.seed_lattice)
    lp = mvn().mvn_prefix_finalize(M, S, cfg.NR).cpu().numpy()
    ls = mvn().mvn_prefix_finalize(Ms, Ss, cfg.NR).cpu().numpy()
    assert np.max(np.abs(lp - ls)) <= 1e-12


def test_units_vs_oracle(torch):
    import test_gpu_parity as P
    from test_parallel_gloo import units_partial
    cfg, T, a = setup(torch, g=13, N=300, R=2, base="A")
    n = cfg.n
    U = mvn().sov_units(cfg.N, cfg.R)
    d_a = torch.from_numpy(a).cuda()
    Pg = mvn().mvn_sov_prefix_units(T, n, d_a, cfg.N, cfg.R, cfg.seed_lattice, 0, U).cpu().numpy()
    L = P.to_dense_lower(T, n)
    Po = units_partial(L, a, cfg.N, cfg.R, cfg.seed_lattice, 0, U)
    for u in range(U):
        cnt = min(128, cfg.NR - 128 * u)
        lg = Pg[u, :, 0] + np.log(Pg[u, :, 1]) - math.log(cnt)
        lo = Po[u, :, 0] + np.log(Po[u, :, 1]) - math.log(cnt)
        assert np.max(np.abs(lg - lo)) <= 1e-11, u


def test_units_combine_forced_nccl(torch):
    """combine_units_deterministic on a one-rank NCCL communicator (all_gather of the padded
    partials forced) equals mvn_prefix_reduce bit for bit."""
    import os
    import torch.distributed as dist
    from paper_2405_14892_b200.parallel import combine_units_deterministic
    from test_gpu_nccl_plumbing import free_port
    if dist.is_initialized():
        pytest.skip("a process group already exists")
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        cfg, T, a = setup(torch, g=15, N=400, R=2, base="A")
        n = cfg.n
        U = mvn().sov_units(cfg.N, cfg.R)
        Pt = mvn().mvn_sov_prefix_units(T, n, torch.from_numpy(a).cuda(), cfg.N, cfg.R, cfg.seed_lattice, 0, U)
        M, S = combine_units_deterministic(Pt, force_collectives=True)
        M1, S1 = mvn().mvn_prefix_reduce(Pt)
        torch.cuda.synchronize()
        assert torch.equal(M, M1) and torch.equal(S, S1)
    finally:
        dist.destroy_process_group()
