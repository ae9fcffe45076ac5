"""NEXT-1 2-D block-cyclic host logic on CPU (gloo, world size 4 as 2 x 2 and 4 x 1, 6 as 3 x 2):
parallel.potrf_distributed_2d — the step loop of potrf_2d_schedule with its collectives (the
diagonal block broadcast in the process-column subgroup, each row block of the super-panel broadcast
from its owner) — run with a numpy stand-in for the libmvn building blocks on 2-D distributed
storage. Every rank's own tiles must be the Cholesky factor of Sigma. The stand-in is test
infrastructure; the product path has no CPU backend."""
import os
import socket

import numpy as np
import pytest
import scipy.linalg as sla
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2405_14892_b200 import parallel

NB = 128


class Numpy2DOps:
    """Owned tiles (I mod P == pr, J mod Q == pc over kp-blocks) as a dict; the panel buffer in the
    kPanel layout as a CPU tensor (the broadcasts move it). Same semantics as mvn_dpotrf_panel (2-D:
    the diagonal block), mvn_dpanel_trsm, mvn_dpanel_pack, mvn_dpotrf_update."""

    def __init__(self, A, P, Q, pr, pc, kp):
        n = A.shape[0]
        self.n, self.nt, self.kp = n, -(-n // NB), kp
        self.P, self.Q, self.pr, self.pc = P, Q, pr, pc
        npad = self.nt * NB
        M = np.eye(npad)
        M[:n, :n] = A
        self.T = {(i, j): M[i * NB:(i + 1) * NB, j * NB:(j + 1) * NB].copy()
                  for i in range(self.nt) for j in range(i + 1) if self.owns(i, j)}
        self.bufs = {}
        self.fail = -1

    def owns(self, i, j):
        return (i // self.kp) % self.P == self.pr and (j // self.kp) % self.Q == self.pc

    def width(self, sp):
        return min(self.kp, self.nt - sp * self.kp)

    def off(self, sp, i):
        k, w = sp * self.kp, self.width(sp)
        m = i - k
        return (m * (m + 1) // 2 if m <= w else w * (w + 1) // 2 + (m - w) * w)

    def panel_buf(self, sp):
        if sp not in self.bufs:
            self.bufs = {sp: torch.zeros(self.off(sp, self.nt) * NB * NB, dtype=torch.float64)}
        return self.bufs[sp]

    def row_block_range(self, sp, I):
        k = sp * self.kp
        lo, hi = max(I * self.kp, k), min((I + 1) * self.kp, self.nt)
        return self.off(sp, lo) * NB * NB, self.off(sp, hi) * NB * NB

    def btile(self, sp, i, c):
        k = sp * self.kp
        o = (self.off(sp, i) + c - k) * NB * NB
        return self.panel_buf(sp)[o:o + NB * NB].numpy().reshape(NB, NB)

    def panel(self, sp, on):                     # the diagonal block (rows of the block only)
        k, w = sp * self.kp, self.width(sp)
        for c in range(k, k + w):
            for i in range(c, k + w):
                for cc in range(k, c):
                    self.T[(i, c)] -= self.T[(i, cc)] @ self.T[(c, cc)].T
            try:
                L = np.linalg.cholesky(self.T[(c, c)])
            except np.linalg.LinAlgError:
                self.fail = c * NB if self.fail < 0 else self.fail
                return
            self.T[(c, c)] = L
            for i in range(c + 1, k + w):
                self.T[(i, c)] = sla.solve_triangular(L, self.T[(i, c)].T, lower=True).T

    def trsm(self, sp, on):                      # own rows below the diagonal block, from the buffer
        k, w = sp * self.kp, self.width(sp)
        for c in range(k, k + w):
            for i in range(k + w, self.nt):
                if not self.owns(i, c):
                    continue
                for cc in range(k, c):
                    self.T[(i, c)] -= self.T[(i, cc)] @ self.btile(sp, c, cc).T
                self.T[(i, c)] = sla.solve_triangular(self.btile(sp, c, c), self.T[(i, c)].T, lower=True).T

    def pack(self, sp, on):
        k, w = sp * self.kp, self.width(sp)
        for i in range(k, self.nt):
            for c in range(k, min(i, k + w - 1) + 1):
                if self.owns(i, c):
                    self.btile(sp, i, c)[:] = self.T[(i, c)]

    def update(self, sp, c0, cs, cb, on, side_busy=True, just_one=None):
        k, w = sp * self.kp, self.width(sp)
        for (i, j), t in self.T.items():
            if j >= c0 and i >= j:
                for c in range(k, k + w):
                    t -= self.btile(sp, i, c) @ self.btile(sp, j, c).T

    def wait(self, h, on):
        pass

    def join(self):
        pass

    def info(self):
        return self.fail


def spd(n, seed=3):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, n))
    return X @ X.T / n + np.eye(n)


def _worker(rank, world, P, port, n, kp, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    Q = world // P
    ops = Numpy2DOps(spd(n), P, Q, rank // Q, rank % Q, kp)
    info = parallel.potrf_distributed_2d(None, n, P, ops=ops)
    out[rank] = (info, {k: v.copy() for k, v in ops.T.items()})
    dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,P,n,kp", [(4, 2, 5 * NB + 17, 1), (4, 4, 6 * NB, 1), (6, 3, 7 * NB + 3, 1),
                                          (4, 2, 9 * NB + 1, 2)])
def test_2d_block_cyclic_schedule_gloo(world, P, n, kp):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, P, free_port(), n, kp, out), nprocs=world, join=True)
    nt = -(-n // NB)
    L = np.linalg.cholesky(spd(n))
    Lp = np.eye(nt * NB)
    Lp[:n, :n] = L
    seen = set()
    for r in range(world):
        info, T = out[r]
        assert info == -1
        for (i, j), t in T.items():
            want = Lp[i * NB:(i + 1) * NB, j * NB:(j + 1) * NB]
            if i == j:
                t, want = np.tril(t), np.tril(want)
            assert np.max(np.abs(t - want)) <= 1e-10, (r, i, j)
            assert (i, j) not in seen
            seen.add((i, j))
    assert len(seen) == nt * (nt + 1) // 2                       # the ranks partition the tiles
