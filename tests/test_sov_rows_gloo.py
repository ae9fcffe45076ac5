"""NEXT-1 sweep over distributed L, host logic on CPU (gloo, world size 2 and 3, 1-D and 2-D storage):
parallel.sov_rows_schedule with its broadcasts — every rank's piece of a phase's tile rows (its owned
tiles of those rows, one contiguous range of its storage, row after row) broadcast from that rank —
driven through a numpy stand-in for the libmvn calls (mvn_drows_unpack, mvn_sweep_rows). The
stand-in sweep checks that every phase sees exactly the rows of the full matrix, in order, and that
the phases cover all rows. The stand-in is test infrastructure; the product path has no CPU backend."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2405_14892_b200 import parallel

NB = 8                                           # small tiles: the schedule does not depend on the size


class NumpySovRowsOps:
    def __init__(self, A, world, rank, kp, P, phases):
        self.nt = A.shape[0] // NB
        self.A, self.world, self.rank, self.kp, self.P, self.phases = A, world, rank, kp, P, phases
        self.Q = world // P
        # this rank's storage: its owned tiles, row after row, columns ascending (mvn_dtiles layout)
        self.local = torch.from_numpy(np.concatenate(
            [self.tile(i, j).ravel() for i in range(self.nt) for j in range(i + 1) if self.owns(rank, i, j)]
            or [np.zeros(0)]))
        mx = max(self.off(r, e) - self.off(r, b) for r in range(world) for b, e in phases)
        self.recv = {r: torch.full((mx,), float("nan"), dtype=torch.float64) for r in range(world) if r != rank}
        self.seen = []

    def tile(self, i, j):
        return self.A[i * NB:(i + 1) * NB, j * NB:(j + 1) * NB]

    def owns(self, r, i, j):
        pr, pc = r // self.Q, r % self.Q
        return (j // self.kp) % self.Q == pc and (i // self.kp) % self.P == pr

    def owned(self, r, b, e):
        return [(i, j) for i in range(b, e) for j in range(i + 1) if self.owns(r, i, j)]

    def off(self, r, i):                          # mvn_drows_offset
        return len(self.owned(r, 0, i)) * NB * NB

    def piece(self, r, p):
        b, e = self.phases[p]
        lo, hi = self.off(r, b), self.off(r, e)
        return self.local[lo:hi] if r == self.rank else self.recv[r][:hi - lo]   # one receive buffer per rank

    def comm(self, p):
        hs = []
        for r in range(self.world):
            buf = self.piece(r, p)
            if buf.numel():
                hs.append(dist.broadcast(buf, src=r, async_op=True))
        return hs

    def wait(self, hs):
        for h in hs or ():
            h.wait()

    def assemble(self, p):                        # mvn_drows_unpack of every rank's piece
        b, e = self.phases[p]
        self.rows = {}
        for r in range(self.world):
            buf = self.piece(r, p).numpy()
            for t, (i, j) in enumerate(self.owned(r, b, e)):
                assert (i, j) not in self.rows
                self.rows[(i, j)] = buf[t * NB * NB:(t + 1) * NB * NB].reshape(NB, NB).copy()

    def sweep(self, p):                           # mvn_sweep_rows: must see exactly rows [b, e)
        b, e = self.phases[p]
        assert sorted(self.rows) == [(i, j) for i in range(b, e) for j in range(i + 1)]
        for (i, j), T in self.rows.items():
            assert np.array_equal(T, self.tile(i, j)), (i, j)
        self.seen.append((b, e))


def _worker(rank, world, port, P, kp, nt, phase_rows, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A = np.random.default_rng(7).normal(size=(nt * NB, nt * NB))
        phases = parallel.sov_phases(nt, phase_rows)
        ops = NumpySovRowsOps(A, world, rank, kp, P, phases)
        parallel.sov_rows_schedule(ops, len(phases))
        assert ops.seen == phases
        assert phases[0][0] == 0 and phases[-1][1] == nt
        assert all(a[1] == b[0] for a, b in zip(phases, phases[1:]))
        q.put((rank, "ok"))
    except Exception as ex:                       # noqa: BLE001
        q.put((rank, repr(ex)))
    finally:
        dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,P,kp,nt,phase_rows", [(2, 1, 2, 9, 2), (3, 1, 1, 7, 3), (2, 2, 2, 8, 1),
                                                      (3, 1, 3, 10, 4), (2, 1, 2, 5, 5)])
def test_sov_rows_schedule_gloo(world, P, kp, nt, phase_rows):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, P, kp, nt, phase_rows, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res


def test_sov_phases():
    assert parallel.sov_phases(10, 4) == [(0, 4), (4, 8), (8, 10)]
    assert parallel.sov_phases(3, 8) == [(0, 3)]
    assert parallel.sov_phases(5, 1) == [(i, i + 1) for i in range(5)]
    assert parallel.sov_phases(0, 3) == []
