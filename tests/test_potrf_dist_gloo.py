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
    semantics as mvn_potrf_panel / mvn_potrf_update / mvn_panel_pack / mvn_panel_unpack with
    super-panels of kp tile columns. `applied[(i, j)]` logs the columns applied to tile (i, j)."""

    def __init__(self, A: np.ndarray, kp: int = 2):
        n = A.shape[0]
        self.n, self.nt, self.kp = n, -(-n // NB), kp
        npad = self.nt * NB
        P = np.eye(npad)
        P[:n, :n] = A
        self.T = np.zeros((self.nt * (self.nt + 1) // 2, NB, NB))
        for i in range(self.nt):
            for j in range(i + 1):
                self.T[tidx(i, j)] = P[i * NB:(i + 1) * NB, j * NB:(j + 1) * NB]
        self.bufs = [np.zeros((kp * self.nt, NB, NB)) for _ in range(2)]
        self.first_fail = -1
        self.log = []
        self.applied = {}

    def cols(self, sp):
        k = sp * self.kp
        return list(range(k, min(k + self.kp, self.nt)))

    def tiles_of(self, sp):
        return [(i, c) for c in self.cols(sp) for i in range(c, self.nt)]

    def panel_buf(self, sp):
        return torch.from_numpy(self.bufs[sp & 1][:len(self.tiles_of(sp))])

    def _apply(self, i, j, cs):
        for c in cs:
            self.T[tidx(i, j)] -= self.T[tidx(i, c)] @ self.T[tidx(j, c)].T
        self.applied.setdefault((i, j), []).extend(cs)

    def panel(self, sp, on):
        cs = self.cols(sp)
        self.log.append(("panel", sp, on))
        for q, c in enumerate(cs):
            for i in range(c, self.nt):
                if q:
                    self._apply(i, c, cs[:q])
            D = self.T[tidx(c, c)]
            try:
                Lcc = np.linalg.cholesky(D)
            except np.linalg.LinAlgError:
                if self.first_fail < 0:
                    self.first_fail = c * NB
                return
            self.T[tidx(c, c)] = Lcc
            for i in range(c + 1, self.nt):
                self.T[tidx(i, c)] = sla.solve_triangular(Lcc, self.T[tidx(i, c)].T, lower=True).T

    def pack(self, sp, on):
        for q, (i, c) in enumerate(self.tiles_of(sp)):
            self.bufs[sp & 1][q] = self.T[tidx(i, c)]

    def unpack(self, sp, on):
        for q, (i, c) in enumerate(self.tiles_of(sp)):
            self.T[tidx(i, c)] = self.bufs[sp & 1][q]

    def update(self, sp, c0, cs, cb, on, side_busy=True):
        self.log.append(("update", sp, c0, cs, cb, on))
        m = 0
        while True:
            base = c0 + m * cs
            if base >= self.nt:
                break
            for b in range(cb):
                j = base + b
                if j < self.nt:
                    for i in range(j, self.nt):
                        self._apply(i, j, self.cols(sp))
            m += 1

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
        for sp in range(20):
            for r in range(world):
                f = owned_first(sp, r, world)
                assert f >= sp and f % world == r and f - sp < world


@pytest.mark.parametrize("world,kp", [(1, 2), (2, 2), (3, 2), (5, 2), (3, 1), (2, 3)])
def test_schedule_covers_every_update_once(world, kp):
    """Replays each rank's schedule: every tile (i, j) of a column the rank owns receives the
    updates of columns 0 .. j-1 exactly once, in ascending order, before column j is factored;
    super-panels are factored by their owners, in order."""
    n = 9 * NB + 17
    nt = -(-n // NB)
    for r in range(world):
        ops = NumpyPotrfOps(np.eye(n), kp)
        for _ in potrf_dist_schedule(ops, r, world):
            pass
        owned_sp = [sp for sp in range(-(-nt // kp)) if sp % world == r]
        assert [e[1] for e in ops.log if e[0] == "panel"] == owned_sp
        for sp in owned_sp:
            for j in ops.cols(sp):
                for i in range(j, nt):
                    assert ops.applied.get((i, j), []) == list(range(j)), (r, i, j, ops.applied.get((i, j)))
        for (i, j), cs in ops.applied.items():
            assert (j // kp) % world == r                     # only own columns are touched


def _worker(rank, world, port, n, out, bad_row):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    A = spd(n)
    if bad_row is not None:
        A[bad_row, bad_row] = -1.0
    ops = NumpyPotrfOps(A, 2)
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
    n, world = 6 * NB, 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, free_port(), n, out, 2 * NB + 5), nprocs=world, join=True)
    # the numpy stand-in reports the first failing tile's first row; both ranks agree on it
    assert out[0][0] == out[1][0] == 2 * NB
