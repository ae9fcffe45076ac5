"""The multi-rank step logic of parallel.crd_step (the north_star layout "rank 0
factors Sigma and broadcasts L, samples shard over the ranks, the per-prefix sums are combined",
and the NEXT-1 layouts "the ranks factor Sigma together", also on distributed storage with the
sweep gathering each phase's rows from the ranks) on CPU with gloo at world size 2 and 3.
The CUDA building blocks are replaced by host stand-ins built on the oracle (test infrastructure;
the product path has no CPU backend); the collectives, the sharding, the ownership of every stage
and the combine are the product code. Every rank must end with the single-process estimate."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import workloads as W
from paper_2405_14892_b200 import parallel


class HostCrdOps:
    """Stand-ins with crd_step's calling conventions. L is a flat CPU tensor holding the dense
    lower factor (row-major n x n); calls are counted per stage."""

    def __init__(self):
        self.calls = {"cov": 0, "potrf": 0, "potrf_dist": 0, "sov": 0}
        self.xy = None

    def cov(self, d_xy, cfg, L):
        import oracle
        self.calls["cov"] += 1
        n = d_xy.shape[0]
        L.copy_(torch.from_numpy(oracle.covariance(d_xy.numpy(), cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget).ravel()))
        assert L.numel() == n * n

    def potrf(self, L, n):
        import oracle
        self.calls["potrf"] += 1
        Lo, info = oracle.cholesky(L.view(n, n).numpy())
        L.copy_(torch.from_numpy(Lo.ravel()))
        return info

    def potrf_dist(self, L, n, group):
        from test_potrf_dist_gloo import NumpyPotrfOps
        self.calls["potrf_dist"] += 1
        ops = NumpyPotrfOps(L.view(n, n).numpy().copy(), kp=1)
        info = parallel.potrf_distributed(L, n, group, ops=ops)
        L.copy_(torch.from_numpy(ops.dense_L().ravel()))
        return info

    def sov(self, L, n, d_a, cfg, begin, end):
        from test_parallel_gloo import range_partial
        self.calls["sov"] += 1
        M, S = range_partial(L.view(n, n).numpy(), d_a.numpy(), cfg.N, cfg.R, cfg.seed_lattice, begin, end)
        return torch.from_numpy(M.copy()), torch.from_numpy(S.copy())

    # potrf="dstore": `L` stands for this rank's storage (the dense matrix here); the factorisation
    # is the distributed schedule; the sweep gathers every phase's rows from the ranks' pieces (the
    # owned tiles of those rows, broadcast over gloo) and runs on the assembled factor
    def dcov(self, d_xy, cfg, L, n, world, rank, kp):
        self.cov(d_xy, cfg, L)

    def potrf_dstore(self, L, n, group, kp):
        return self.potrf_dist(L, n, group)

    def sov_dstore(self, L, n, d_a, cfg, begin, end, kp, group):
        from test_sov_rows_gloo import NB, NumpySovRowsOps
        self.calls["sov"] += 1
        world, rank = dist.get_world_size(), dist.get_rank()
        npad = -(-n // NB) * NB
        A = np.eye(npad)
        A[:n, :n] = np.tril(L.view(n, n).numpy())
        phases = parallel.sov_phases(npad // NB, 3)
        ops = NumpySovRowsOps(A, world, rank, kp, 1, phases)
        got = np.full((npad, npad), np.nan)
        sweep = ops.sweep

        def record(p):                            # the stand-in sweep: keep the phase's rows
            sweep(p)
            for (i, j), T in ops.rows.items():
                got[i * NB:(i + 1) * NB, j * NB:(j + 1) * NB] = T
        ops.sweep = record
        parallel.sov_rows_schedule(ops, len(phases))
        Lg = np.tril(got)[:n, :n]
        assert not np.isnan(Lg).any()
        from test_parallel_gloo import range_partial
        M, S = range_partial(Lg, d_a.numpy(), cfg.N, cfg.R, cfg.seed_lattice, begin, end)
        return torch.from_numpy(M.copy()), torch.from_numpy(S.copy())

    @staticmethod
    def rescale(Mg, M, S):
        from test_parallel_gloo import torch_rescale
        torch_rescale(Mg, M, S)

    @staticmethod
    def finalize(M, S, NR):
        return M + torch.log(S) - math.log(NR)


def problem():
    import oracle
    cfg = W.small_config("crd-gloo", 15, 200, 3, base="C")       # n = 225 (two tiles), nu = 3/2, u = 0.5
    inp = W.make_inputs(cfg)
    order, a, _ = oracle.marginal_order(inp.mu, np.full(cfg.n, cfg.sigma2 + cfg.nugget), cfg.u)
    return cfg, inp, order, a


def _worker(rank, world, port, mode, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg, inp, order, a = problem()
    n = cfg.n
    ops = HostCrdOps()
    L = torch.full((n * n,), float("nan"), dtype=torch.float64)    # only what the step writes is valid
    logp = parallel.crd_step(torch.from_numpy(np.ascontiguousarray(inp.xy[order])), torch.from_numpy(a), L, cfg,
                             potrf=mode, ops=ops)
    out[rank] = (logp.numpy().copy(), L.numpy().copy(), dict(ops.calls))
    dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("mode", ["rank0", "dist", "auto", "dstore"])
def test_crd_step_multi_rank_matches_single_process(world, mode):
    import oracle
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, free_port(), mode, out), nprocs=world, join=True)
    cfg, inp, order, a = problem()
    ref = oracle.crd(inp.xy, inp.mu, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget, cfg.u, cfg.N, cfg.R,
                     cfg.seed_lattice, cfg.conf, chunk=cfg.N)
    for r in range(world):
        lp, L, calls = out[r]
        assert np.max(np.abs(lp - ref.logp)) <= 1e-12, (r, np.max(np.abs(lp - ref.logp)))
        assert np.array_equal(L, out[0][1])                          # every rank holds the same L
        assert calls["sov"] == 1
        if mode in ("dist", "dstore"):
            assert calls["cov"] == 1 and calls["potrf_dist"] == 1 and calls["potrf"] == 0
        else:                                                        # auto = rank0: the north_star layout
            assert calls["potrf_dist"] == 0
            assert (calls["cov"], calls["potrf"]) == ((1, 1) if r == 0 else (0, 0))
    assert np.array_equal(out[0][0], out[world - 1][0])              # same log P on every rank
    k0, _ = oracle.region(out[0][0], cfg.conf)
    assert np.array_equal(k0, ref.k_star)
