"""Multi-GPU plumbing (torch.distributed, NCCL over NVLink/NVSwitch): SURVEY §8(e), DESIGN.md §7.

Given L, every QMC sample is independent ("parallel only across MC chains"), so the sweep
shards over samples with no data-path collective inside the kernels:
  * rank 0 generates Sigma and factors it (north_star), then broadcast(L) from rank 0 (C1);
  * rank g sweeps its contiguous global sample range [g*NR/W, (g+1)*NR/W) — with N*R = 80,000 at
    8 GPUs this is one lattice shift per rank (config D);
  * per-prefix (M_k, S_k): all_reduce(MAX) on M (C2), S <- S exp(M - Mglob) (mvn_prefix_rescale),
    all_reduce(SUM) on S (C3); log P_k = M_k + log S_k - log(NR) on every rank.
The combine is written against an injectable `rescale` so the host logic is testable on CPU with
gloo (tests/test_parallel_gloo.py); on the GPU path it is the CUDA kernel behind mvn_prefix_rescale.

NEXT-1: `potrf_distributed` factors Sigma across the ranks instead of on
rank 0 alone — 1-D block-cyclic over 128-wide tile columns (column j owned by rank j mod W), one
step of lookahead, the finished panel of each step broadcast over NCCL while the ranks update
their own columns. Every rank ends with all of L, so the broadcast of L (C1) disappears.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Balanced contiguous split of [0, total) into `world` ranges; rank's [begin, end)."""
    if world < 1 or not (0 <= rank < world) or total < world:
        raise ValueError(f"cannot shard {total} samples over {world} ranks")
    base, rem = divmod(total, world)
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


def combine_prefix(M: torch.Tensor, S: torch.Tensor, group=None, rescale=None) -> tuple[torch.Tensor, torch.Tensor]:
    """In place: M <- max over ranks, S <- sum over ranks of S_g exp(M_g - Mglob). Returns (M, S)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return M, S
    Mg = M.clone()
    dist.all_reduce(Mg, op=dist.ReduceOp.MAX, group=group)
    if rescale is None:
        from . import mvn_prefix_rescale as rescale
    rescale(Mg, M, S)
    dist.all_reduce(S, op=dist.ReduceOp.SUM, group=group)
    return M, S


def broadcast_L(L: torch.Tensor, group=None, src: int = 0) -> torch.Tensor:
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.broadcast(L, src=src, group=group)
    return L


def crd_step(d_xy_sorted: torch.Tensor, d_a: torch.Tensor, L: torch.Tensor, cfg, group=None, events=None,
             potrf: str = "auto"):
    """One pass of the whole hot path (a2..a9) on this rank; returns device log P (n,).

    potrf: "rank0" — rank 0 builds and factors Sigma, then broadcasts L (C1, the north_star
    layout); "dist" — every rank builds Sigma and the ranks factor it together
    (potrf_distributed, NEXT-1), after which every rank holds L; "auto" = "dist" when W > 1.
    events: optional list to which (name, event) pairs are appended for stage timing.
    """
    from . import mvn_cov_matern, mvn_potrf, mvn_sov_prefix, mvn_prefix_finalize
    n = d_a.numel()
    world = dist.get_world_size(group) if (dist.is_available() and dist.is_initialized()) else 1
    rank = dist.get_rank(group) if world > 1 else 0
    mode = ("dist" if world > 1 else "rank0") if potrf == "auto" else potrf

    def mark(name):
        if events is None:
            return None
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        events.append((name, e))
        return e

    mark("start")
    if mode == "dist":
        mvn_cov_matern(d_xy_sorted, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget, out=L)
        mark("cov")
        info = potrf_distributed(L, n, group)
        if info != -1:
            raise FloatingPointError(f"Sigma not SPD at row {info}")
        mark("potrf")
        mark("bcast")
    else:
        if rank == 0:
            mvn_cov_matern(d_xy_sorted, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget, out=L)
            mark("cov")
            info = mvn_potrf(L, n)
            if info != -1:
                raise FloatingPointError(f"Sigma not SPD at row {info}")
            mark("potrf")
        else:
            mark("cov")
            mark("potrf")
        broadcast_L(L, group)
        mark("bcast")
    begin, end = shard_range(cfg.N * cfg.R, rank, world)
    M, S = mvn_sov_prefix(L, n, d_a, cfg.N, cfg.R, cfg.seed_lattice, begin, end)
    mark("sov")
    combine_prefix(M, S, group)
    mark("combine")
    logp = mvn_prefix_finalize(M, S, cfg.N * cfg.R)
    mark("finalize")
    return logp


def potrf_launches(n: int, world: int = 1, rank: int = 0, nsm: int = 148) -> int:
    """Kernels launched by one factorisation: mvn_potrf (world 1) or this rank's share of
    potrf_distributed (panel = POTRF + TRSM, update, pack / unpack)."""
    nt = -(-n // TILE)
    if world == 1:
        c = 1 + (1 if nt > 1 else 0)
        for k in range(nt - 1):
            T = nt - k - 1
            c += (1 if T > 1 else 0) + 1 + 1 + (1 if T > 1 else 0)
        return c
    c = 0
    for k in range(nt):
        if k % world == rank:
            c += 1 + (1 if k + 1 < nt else 0) + 1         # panel (potrf [+ trsm]) + pack
        else:
            c += 1                                        # unpack
        if k + 1 < nt:
            if (k + 1) % world == rank:
                c += 1                                    # lookahead column update
            first = owned_first(k + 1, rank, world)
            if first == k + 1 and (k + 1) % world == rank:
                first += world
            c += 1 if first < nt else 0
    return c


# ------------------------------------------------------------------------------------- NEXT-1
TILE = 128


def owned_first(col: int, rank: int, world: int) -> int:
    """Smallest tile column >= col owned by `rank` under the 1-D block-cyclic map j -> j mod world."""
    return col + ((rank - col) % world)


def potrf_dist_schedule(ops, rank: int, world: int):
    """The per-rank step loop of the distributed right-looking Cholesky, as a generator.

    It yields ("bcast", k, src) whenever panel k (tile column k, packed into ops.panel_buf(k)) must
    be broadcast from rank src, and is resumed with a handle that `ops.wait` understands. Runners:
    `potrf_distributed` (torch.distributed, one generator per process) and the single-device
    emulator in the tests (W generators stepped in lockstep). The recurrence is mvn_potrf's
    (Alg. 1 l.8); only the ownership of the updates is split:
      panel k   : owner(k) = k mod W runs POTRF(A_kk) + TRSM(A_ik) and packs the column;
      lookahead : owner(k+1) updates column k+1 with panel k and factors panel k+1 on the side
                  stream, whose broadcast then overlaps the bulk update of step k;
      bulk      : every rank updates its own columns >= k+1 (minus the lookahead column).
    """
    nt = ops.nt
    owner = lambda k: k % world
    if rank == owner(0):
        ops.panel(0, "side")
        ops.pack(0, "side")
    h = yield ("bcast", 0, owner(0))
    for k in range(nt):
        ops.wait(h, "main")                      # panel k has arrived (or was produced here)
        if rank != owner(k):
            ops.unpack(k, "main")
        ev = ops.record("main")                  # also orders every earlier bulk update
        if k + 1 < nt:
            ops.wait(ev, "side")
            if rank == owner(k + 1):
                ops.update(k, k + 1, nt, "side")                 # column k+1 only
                ops.panel(k + 1, "side")
                ops.pack(k + 1, "side")
            h = yield ("bcast", k + 1, owner(k + 1))
            first = owned_first(k + 1, rank, world)
            if first == k + 1 and rank == owner(k + 1):
                first += world
            ops.update(k, first, world, "main", side_busy=(rank == owner(k + 1)))
    ops.join()


class CudaPotrfOps:
    """libmvn building blocks for potrf_dist_schedule on one device: the bulk updates on `main`
    (default: torch's current stream), the panel chain on a high-priority side stream."""

    SIDE_SMS = 8                                 # SMs left free for the panel chain (cf. kPanelSMs)

    def __init__(self, L, n: int, main=None):
        import torch
        from . import panel_numel
        self.torch = torch
        self.L, self.n = L, n
        self.nt = -(-n // TILE)
        self.dev = L.device
        self.main = main if main is not None else torch.cuda.current_stream(self.dev)
        self.side = torch.cuda.Stream(device=self.dev, priority=-1)
        self.side.wait_stream(self.main)
        m = panel_numel(n, 0)
        self.bufs = [torch.empty(m, dtype=torch.float64, device=self.dev) for _ in range(2)]

    def _st(self, which):
        return self.main if which == "main" else self.side

    def panel_buf(self, k: int):
        from . import panel_numel
        return self.bufs[k & 1][:panel_numel(self.n, k)]

    def panel(self, k, on):
        from . import mvn_potrf_panel
        mvn_potrf_panel(self.L, self.n, k, stream=self._st(on))

    def pack(self, k, on):
        from . import mvn_panel_pack
        mvn_panel_pack(self.L, self.n, k, self.panel_buf(k), stream=self._st(on))

    def unpack(self, k, on):
        from . import mvn_panel_unpack
        mvn_panel_unpack(self.panel_buf(k), self.n, k, self.L, stream=self._st(on))

    def update(self, k, c0, cs, on, side_busy=True):
        from . import mvn_potrf_update
        if c0 < self.nt:
            reserve = self.SIDE_SMS if (on == "main" and side_busy) else 0
            mvn_potrf_update(self.L, self.n, k, c0, cs, reserve, stream=self._st(on))

    def record(self, on):
        ev = self.torch.cuda.Event()
        ev.record(self._st(on))
        return ev

    def wait(self, h, on):
        """h: None (nothing to wait for), a torch.cuda.Event, or a torch.distributed Work."""
        if h is None:
            return
        st = self._st(on)
        if isinstance(h, self.torch.cuda.Event):
            st.wait_event(h)
        else:
            with self.torch.cuda.stream(st):
                h.wait()

    def join(self):
        self.main.wait_stream(self.side)


def potrf_distributed(L, n: int, group=None, ops=None) -> int:
    """Distributed tiled Cholesky of the tile-packed Sigma in `L` (every rank holds the full buffer
    with the same Sigma); on return every rank's `L` holds all of L. Returns info (-1 = SPD, else
    the first failing 0-based row, agreed over the ranks). With one rank this is the lookahead
    schedule of mvn_potrf driven from Python."""
    world = dist.get_world_size(group) if (dist.is_available() and dist.is_initialized()) else 1
    rank = dist.get_rank(group) if world > 1 else 0
    if ops is None:
        _cuda_info(L)                            # reset the device pivot flag (synchronises)
        ops = CudaPotrfOps(L, n)
    gen = potrf_dist_schedule(ops, rank, world)
    req = next(gen, None)
    while req is not None:
        _, k, src = req
        h = None
        if world == 1:
            h = ops.record("side")               # the panel chain ran on the side stream
        else:
            buf = ops.panel_buf(k)
            if getattr(ops, "side", None) is not None:
                with torch.cuda.stream(ops.side):
                    h = dist.broadcast(buf, src=dist.get_global_rank(group, src) if group is not None else src,
                                       group=group, async_op=True)
            else:
                dist.broadcast(buf, src=src, group=group)
        try:
            req = gen.send(h)
        except StopIteration:
            req = None
    info = ops.info() if hasattr(ops, "info") else _cuda_info(L)
    if world > 1:
        big = 1 << 62
        t = torch.tensor([info if info >= 0 else big], dtype=torch.int64, device=getattr(ops, "dev", "cpu"))
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
        info = int(t.item())
        info = -1 if info == big else info
    return info


def _cuda_info(L) -> int:
    from . import mvn_potrf_info
    return mvn_potrf_info(L.device.index, reset=True)
