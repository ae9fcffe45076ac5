"""The multi-GPU plumbing on a real NCCL communicator, on the one GPU this pool provides: a one-rank
NCCL process group drives potrf_distributed with its broadcasts forced (async NCCL broadcast issued
from the side stream, Work.wait on the main stream, info all_reduce) and combine_prefix with its
all_reduces forced. Results must equal the single-GPU calls bit for bit. No ranks wait on each
other (world size 1): this checks the stream / event / NCCL ordering the 8-GPU run relies on."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl(cuda_device):
    import torch
    import torch.distributed as dist
    if dist.is_initialized():
        pytest.skip("a process group already exists")
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


def test_potrf_distributed_with_nccl_broadcasts(nccl):
    import torch
    import paper_2405_14892_b200 as mvn
    from paper_2405_14892_b200.parallel import potrf_distributed
    for n in (900, 40 * 128 + 77):
        xy = np.random.default_rng(n).uniform(size=(n, 2))
        T = mvn.mvn_cov_matern(torch.from_numpy(xy).cuda(), 1.0, 0.1, 0.5, 1e-8)
        ref = T.clone()
        assert mvn.mvn_potrf(ref, n) == -1
        assert potrf_distributed(T, n, force_collectives=True) == -1
        torch.cuda.synchronize()
        assert torch.equal(T, ref)


def test_combine_prefix_with_nccl_allreduce(nccl):
    import torch
    import paper_2405_14892_b200 as mvn
    from paper_2405_14892_b200.parallel import combine_prefix
    import workloads as W
    cfg = W.small_config("nccl", 15, 500, 2)
    inp = W.make_inputs(cfg)
    n = cfg.n
    order, a, _ = mvn.mvn_marginal_order(inp.mu, np.full(n, cfg.sigma2 + cfg.nugget), cfg.u)
    T = mvn.mvn_cov_matern(torch.from_numpy(np.ascontiguousarray(inp.xy[order])).cuda(), cfg.sigma2, cfg.beta, cfg.nu,
                           cfg.nugget)
    mvn.mvn_potrf(T, n)
    d_a = torch.from_numpy(a).cuda()
    M, S = mvn.mvn_sov_prefix(T, n, d_a, cfg.N, cfg.R, cfg.seed_lattice)
    M2, S2 = M.clone(), S.clone()
    combine_prefix(M2, S2, force_collectives=True)
    torch.cuda.synchronize()
    assert torch.equal(M2, M) and torch.equal(S2, S)


@pytest.mark.parametrize("mode", ["rank0", "dist", "dstore"])
def test_crd_step_with_nccl_collectives_equals_mvn_crd(nccl, mode):
    """The multi-GPU step (parallel.crd_step) on the one-rank NCCL communicator with every
    collective forced — broadcast_L of the whole tile buffer (rank0, the north_star C1), or the
    distributed Cholesky's panel broadcasts (dist, NEXT-1), or distributed storage end to end with
    the sweep's phase broadcasts (dstore, NEXT-1), then the all_reduce combine — returns
    log P bitwise equal to the single-GPU C call mvn_crd on the same inputs."""
    import torch
    import paper_2405_14892_b200 as mvn
    from paper_2405_14892_b200 import parallel
    import workloads as W
    cfg = W.small_config("nccl-crd", 30, 1000, 3, base="C")        # n = 900, nu = 3/2
    inp = W.make_inputs(cfg)
    n = cfg.n
    ref = mvn.mvn_crd(inp.xy, inp.mu, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget, cfg.u, cfg.N, cfg.R,
                      cfg.seed_lattice, cfg.conf)
    order, a, _ = mvn.mvn_marginal_order(inp.mu, np.full(n, cfg.sigma2 + cfg.nugget), cfg.u)
    d_xy = torch.from_numpy(np.ascontiguousarray(inp.xy[order])).cuda()
    d_a = torch.from_numpy(a).cuda()
    L = mvn.alloc_dtiles(n, 1, 0, mvn.mvn_potrf_panel_width(n)) if mode == "dstore" else mvn.alloc_tiles(n)
    parallel.FORCE_COLLECTIVES = True
    try:
        ev = []
        lp = parallel.crd_step(d_xy, d_a, L, cfg, potrf=mode, events=ev).cpu().numpy()
    finally:
        parallel.FORCE_COLLECTIVES = False
    assert [e[0] for e in ev] == ["start", "cov", "potrf", "bcast", "sov", "combine", "finalize"]
    assert np.array_equal(lp, ref.logP)
    k, _ = mvn.mvn_confidence_region(lp, cfg.conf)
    assert np.array_equal(k, ref.k_star)


def test_broadcast_L_forced_is_identity(nccl):
    import torch
    import paper_2405_14892_b200 as mvn
    from paper_2405_14892_b200.parallel import broadcast_L
    n = 700
    T = mvn.mvn_cov_matern(torch.from_numpy(np.random.default_rng(2).uniform(size=(n, 2))).cuda(), 1.0, 0.1, 0.5, 1e-8)
    T0 = T.clone()
    broadcast_L(T, force_collectives=True)
    torch.cuda.synchronize()
    assert torch.equal(T, T0)


def test_sov_distributed_with_nccl_broadcasts(nccl):
    """The sweep over distributed L (NEXT-1) on the one-rank NCCL communicator with the phase
    broadcasts forced (issued asynchronously before the previous phase's sweep, waited on before
    the assembly): (M, S) bitwise equal to mvn_sov_prefix on the same factor."""
    import torch
    import paper_2405_14892_b200 as mvn
    from paper_2405_14892_b200.parallel import sov_distributed
    n = 40 * 128 + 77
    xy = np.random.default_rng(4).uniform(size=(n, 2))
    d_xy = torch.from_numpy(xy).cuda()
    kp = mvn.mvn_potrf_panel_width(n)
    loc = mvn.alloc_dtiles(n, 1, 0, kp)
    L = mvn.mvn_cov_matern(d_xy, 1.0, 0.05, 1.5, 1e-8)
    assert mvn.mvn_potrf(L, n) == -1
    assert loc.numel() == L.numel()             # W = 1: the local layout is the full tile-packed one
    loc.copy_(L)
    a = torch.from_numpy(np.random.default_rng(5).normal(0.3, 1.0, n)).cuda()
    M, S = sov_distributed(loc, n, a, 2000, 3, 7, 100, 5900, kp, phase_rows=6, force_collectives=True)
    M0, S0 = mvn.mvn_sov_prefix(L, n, a, 2000, 3, 7, 100, 5900)
    torch.cuda.synchronize()
    assert torch.equal(M, M0) and torch.equal(S, S0)
