"""NEXT-1 host logic on CPU (gloo, world_size 2 and 3): the distributed Cholesky schedule
(paper_2405_14892_b200.parallel.potrf_dist_schedule / potrf_distributed — 1-D block-cyclic tile
columns, lookahead, panel broadcasts) run with a numpy stand-in for the five libmvn building
blocks. Every rank must end with the complete factor of Sigma and the same info. The stand-in
is test infrastructure: the product path has no CPU backend."""
import os
import socket

import numpy as np
import pytest
import scipy.linalg as sla
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2405_14892_b200.parallel import owned_first, potrf_dist_schedule, potrf_distributed

NB = 128


def tidx(i, j):
    return i * (i + 1) // 2 + j


class NumpyPotrfOps:
    """Tile-packed lower storage as an array [tiles][nb][nb] (logical row-major tiles); the same
    semantics as mvn_potrf_panel / mvn_potrf_update / mvn_panel_pack / mvn_panel_unpack."""

    def __init__(self, A: np.ndarray):
        n = A.shape[0]
        self.n, self.nt = n, -(-n // NB)
        npad = self.nt * NB
        P = np.eye(npad)
        P[:n, :n] = A
        self.T = np.zeros((self.nt * (self.nt + 1) // 2, NB, NB))
        for i in range(self.nt):
            for j in range(i + 1):
                self.T[tidx(i, j)] = P[i * NB:(i + 1) * NB, j * NB:(j + 1) * NB]
        self.bufs = [np.zeros((self.nt, NB, NB)) for _ in range(2)]
        self.first_fail = -1
        self.log = []

    def panel_buf(self, k):
        return torch.from_numpy(self.bufs[k & 1][:self.nt - k])

    def panel(self, k, on):
        self.log.append(("panel", k, on))
        D = self.T[tidx(k, k)]
        try:
            Lkk = np.linalg.cholesky(D)
        except np.linalg.LinAlgError:
            if self.first_fail < 0:
                d = np.linalg.eigvalsh(D)
                self.first_fail = k * NB
            return
        self.T[tidx(k, k)] = Lkk
        for i in range(k + 1, self.nt):
            self.T[tidx(i, k)] = sla.solve_triangular(Lkk, self.T[tidx(i, k)].T, lower=True).T

    def pack(self, k, on):
        for i in range(k, self.nt):
            self.bufs[k & 1][i - k] = self.T[tidx(i, k)]

    def unpack(self, k, on):
        for i in range(k, self.nt):
            self.T[tidx(i, k)] = self.bufs[k & 1][i - k]

    def update(self, k, c0, cs, on, side_busy=True):
        self.log.append(("update", k, c0, cs, on))
        for j in range(c0, self.nt, cs):
            for i in range(j, self.nt):
                self.T[tidx(i, j)] -= self.T[tidx(i, k)] @ self.T[tidx(j, k)].T

    def record(self, on):
        return None

    def wait(self, h, on):
        pass

    def join(self):
        pass

    def info(self):
        return self.first_fail

    def dense_L(self):
        P = np.zeros((self.nt * NB, self.nt * NB))
        for i in range(self.nt):
            for j in range(i + 1):
                P[i * NB:(i + 1) * NB, j * NB:(j + 1) * NB] = self.T[tidx(i, j)]
        return np.tril(P)[:self.n, :self.n]


def spd(n, seed=3):
    rng = np.random.default_rng(seed)
    xy = rng.uniform(size=(n, 2))
    h = np.sqrt(((xy[:, None, :] - xy[None, :, :]) ** 2).sum(-1))
    return np.exp(-h / 0.2) + 1e-8 * np.eye(n)


def test_owned_first():
    for world in (1, 2, 3, 8):
        for col in range(20):
            for r in range(world):
                f = owned_first(col, r, world)
                assert f >= col and f % world == r and f - col < world


@pytest.mark.parametrize("world", [1, 2, 3, 5])
def test_schedule_covers_every_update_once(world):
    """Replays the schedule of all ranks in lockstep: each tile (i, j) receives the updates of
    panels 0..j-1 exactly once, in ascending k, on the rank that owns column j, before column j
    is factored; panels are factored in order by their owners."""
    n = 9 * NB + 17
    nt = -(-n // NB)
    logs = []
    for r in range(world):
        ops = NumpyPotrfOps(np.eye(n))
        g = potrf_dist_schedule(ops, r, world)
        for _ in g:
            pass
        logs.append(ops.log)
    for r in range(world):
        seen = {}
        factored = set()
        for ev in logs[r]:
            if ev[0] == "panel":
                k = ev[1]
                assert k % world == r
                assert all(seen.get((i, k), []) == list(range(k)) for i in range(k, nt))
                factored.add(k)
            else:
                _, k, c0, cs, _ = ev
                for j in range(c0, nt, cs):
                    assert j % world == r and j > k
                    for i in range(j, nt):
                        seen.setdefault((i, j), []).append(k)
        assert factored == {k for k in range(nt) if k % world == r}


def _worker(rank, world, port, n, out, bad_row):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    A = spd(n)
    if bad_row is not None:
        A[bad_row, bad_row] = -1.0
    ops = NumpyPotrfOps(A)
    info = potrf_distributed(None, n, ops=ops)
    out[rank] = (info, ops.dense_L())
    dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_potrf_gloo(world):
    n = 5 * NB + 40
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, free_port(), n, out, None), nprocs=world, join=True)
    A = spd(n)
    Lref = np.linalg.cholesky(A)
    for r in range(world):
        info, L = out[r]
        assert info == -1
        assert np.max(np.abs(L - Lref)) <= 1e-10
    assert all(np.array_equal(out[0][1], out[r][1]) for r in range(world))


def test_distributed_potrf_gloo_reports_failure():
    n, world = 4 * NB, 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, free_port(), n, out, 2 * NB + 5), nprocs=world, join=True)
    # the numpy stand-in reports the first failing tile's first row; both ranks agree on it
    assert out[0][0] == out[1][0] == 2 * NB
