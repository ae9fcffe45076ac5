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
rank 0 alone — 1-D block-cyclic over super-panels of kp tile columns (super-panel s owned by
rank s mod W), one step of lookahead, the finished panel of each step broadcast over NCCL while the
ranks update their own columns. With a full buffer per rank (CudaPotrfOps) every rank ends with all
of L, so the broadcast of L (C1) disappears; with distributed storage (CudaPotrfDistOps,
potrf_distributed_local) a rank holds only its own columns (~1/W of the memory).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

# Testing aid: issue the collectives of the multi-GPU path even on a one-rank process group
# (bench.py --force-dist), so the NCCL plumbing runs on a single GPU.
FORCE_COLLECTIVES = False


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Balanced contiguous split of [0, total) into `world` ranges; rank's [begin, end)."""
    if world < 1 or not (0 <= rank < world) or total < world:
        raise ValueError(f"cannot shard {total} samples over {world} ranks")
    base, rem = divmod(total, world)
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


def combine_prefix(M: torch.Tensor, S: torch.Tensor, group=None, rescale=None,
                   force_collectives: bool = False) -> tuple[torch.Tensor, torch.Tensor]:
    """In place: M <- max over ranks, S <- sum over ranks of S_g exp(M_g - Mglob). Returns (M, S)."""
    if not (dist.is_available() and dist.is_initialized()):
        return M, S
    if dist.get_world_size(group) == 1 and not (force_collectives or FORCE_COLLECTIVES):
        return M, S
    Mg = M.clone()
    dist.all_reduce(Mg, op=dist.ReduceOp.MAX, group=group)
    if rescale is None:
        from . import mvn_prefix_rescale as rescale
    rescale(Mg, M, S)
    dist.all_reduce(S, op=dist.ReduceOp.SUM, group=group)
    return M, S


def combine_units_deterministic(partial: torch.Tensor, group=None, reduce=None,
                                force_collectives: bool = False) -> tuple[torch.Tensor, torch.Tensor]:
    """SURVEY §8(e)'s bitwise-deterministic combine: every rank holds the per-unit partials
    [units][n][2] of its contiguous unit range (mvn_sov_prefix_units over shard_range(U, rank, W));
    the ranks' ranges are all-gathered (padded to the longest with (-inf, 0) units, which the
    reduction skips) and reduced in global unit order (mvn_prefix_reduce). The result is the same
    bits on every rank and for every W. `reduce` defaults to mvn_prefix_reduce (tests pass a host
    stand-in)."""
    if reduce is None:
        from . import mvn_prefix_reduce as reduce
    if not (dist.is_available() and dist.is_initialized()) or \
            (dist.get_world_size(group) == 1 and not (force_collectives or FORCE_COLLECTIVES)):
        return reduce(partial)
    W = dist.get_world_size(group)
    cnt = torch.tensor([partial.shape[0]], dtype=torch.int64, device=partial.device)
    cnts = [torch.empty_like(cnt) for _ in range(W)]
    dist.all_gather(cnts, cnt, group=group)
    mx = int(max(int(c.item()) for c in cnts))
    pad = torch.empty((mx, partial.shape[1], 2), dtype=partial.dtype, device=partial.device)
    pad[..., 0] = float("-inf")
    pad[..., 1] = 0.0
    pad[:partial.shape[0]] = partial
    parts = [torch.empty_like(pad) for _ in range(W)]
    dist.all_gather(parts, pad, group=group)
    return reduce(torch.cat(parts, 0).contiguous())


def broadcast_L(L: torch.Tensor, group=None, src: int = 0, force_collectives: bool = False) -> torch.Tensor:
    """C1: rank `src` (group rank) sends the tile-packed factor to every rank (NCCL over NVLink), in
    place. A no-op without a process group, and on one rank unless collectives are forced."""
    if not (dist.is_available() and dist.is_initialized()):
        return L
    if dist.get_world_size(group) > 1 or force_collectives or FORCE_COLLECTIVES:
        g_src = dist.get_global_rank(group, src) if group is not None else src
        dist.broadcast(L, src=g_src, group=group)
    return L


class LibmvnCrdOps:
    """The building blocks crd_step drives, on the CUDA library (the product path). Tests replace
    them with host stand-ins to run the multi-rank step logic on CPU with gloo."""

    @staticmethod
    def cov(d_xy, cfg, L):
        from . import mvn_cov_matern
        mvn_cov_matern(d_xy, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget, out=L)

    potrf_method = 0         # 0: fp64 DMMA (default), 1: the trailing updates on the int8 tensor cores,
    tlr_eps = 1e-3           # 2: the TLR Cholesky at accuracy tlr_eps (NEXT-3, R26; slots cached per n)
    _tlr_slots = {}

    @classmethod
    def potrf(cls, L, n):
        from . import mvn_potrf_ex, mvn_tlr_potrf
        if cls.potrf_method == 2:
            key = (L.device.index, n)
            if key not in cls._tlr_slots:
                nt = -(-n // 128)
                noff = max(nt * (nt - 1) // 2, 1)
                cls._tlr_slots.clear()
                cls._tlr_slots[key] = tuple(torch.empty((noff, 128, 128), dtype=torch.float64, device=L.device)
                                            for _ in range(2))
            U, V = cls._tlr_slots[key]
            return mvn_tlr_potrf(L, n, cls.tlr_eps, U=U, V=V).info
        return mvn_potrf_ex(L, n, cls.potrf_method)

    @staticmethod
    def potrf_dist(L, n, group):
        return potrf_distributed(L, n, group)

    sov_method = 0           # 0: fp64 DMMA (default), 1: the GEMM on the int8 tensor cores (NEXT-4)

    @classmethod
    def sov(cls, L, n, d_a, cfg, begin, end):
        from . import mvn_sov_prefix_ex
        return mvn_sov_prefix_ex(L, n, d_a, cfg.N, cfg.R, cfg.seed_lattice, begin, end, method=cls.sov_method)

    # distributed storage end to end (potrf="dstore"): L is this rank's mvn_dtiles buffer
    @staticmethod
    def dcov(d_xy, cfg, local, n, world, rank, kp):
        from . import dtiles, mvn_dcov_matern
        mvn_dcov_matern(d_xy, dtiles(n, world, rank, kp), cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget, local)

    @staticmethod
    def potrf_dstore(local, n, group, kp):
        return potrf_distributed_local(local, n, group, kp=kp)

    phase_rows = 16          # tile rows per phase of the sweep over distributed L

    @classmethod
    def sov_dstore(cls, local, n, d_a, cfg, begin, end, kp, group):
        return sov_distributed(local, n, d_a, cfg.N, cfg.R, cfg.seed_lattice, begin, end, kp, group=group,
                               phase_rows=cls.phase_rows)

    @staticmethod
    def rescale(Mg, M, S):
        from . import mvn_prefix_rescale
        mvn_prefix_rescale(Mg, M, S)

    @staticmethod
    def finalize(M, S, NR):
        from . import mvn_prefix_finalize
        return mvn_prefix_finalize(M, S, NR)


def crd_ops(sov_method: int = 0, potrf_method: int = 0, tlr_eps: float = 1e-3):
    """LibmvnCrdOps with the chosen arithmetic for the SOV GEMM and the Cholesky updates (NEXT-4), or
    the TLR Cholesky (potrf_method 2, NEXT-3)."""
    if sov_method == 0 and potrf_method == 0:
        return LibmvnCrdOps
    return type("LibmvnCrdOpsMixed", (LibmvnCrdOps,), {"sov_method": sov_method, "potrf_method": potrf_method,
                                                       "tlr_eps": tlr_eps})


def crd_step(d_xy_sorted: torch.Tensor, d_a: torch.Tensor, L: torch.Tensor, cfg, group=None, events=None,
             potrf: str = "auto", ops=None):
    """One pass of the whole hot path (a2..a9) on this rank; returns device log P (n,).

    potrf: "rank0" — rank 0 builds and factors Sigma, then broadcasts L (C1, the north_star
    layout); "dist" — every rank builds Sigma and the ranks factor it together
    (potrf_distributed, NEXT-1), after which every rank holds L; "dstore" — NEXT-1 on distributed
    storage end to end: `L` is this rank's mvn_dtiles buffer (1-D, kp = mvn_potrf_panel_width(n),
    ~1/W of the tiles), Sigma generated there, factored by potrf_distributed_local, and the sweep
    gathers each phase's rows from the ranks (sov_distributed); "auto" = "rank0".
    events: optional list to which (name, event) pairs are appended for stage timing.
    ops: the building blocks (default LibmvnCrdOps, the CUDA library).
    """
    ops = ops or LibmvnCrdOps
    n = d_a.numel()
    world = dist.get_world_size(group) if (dist.is_available() and dist.is_initialized()) else 1
    rank = dist.get_rank(group) if world > 1 else 0
    mode = "rank0" if potrf == "auto" else potrf
    if mode not in ("rank0", "dist", "dstore"):
        raise ValueError(f"potrf must be auto, rank0, dist or dstore, not {potrf!r}")

    def mark(name):
        if events is None:
            return None
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        events.append((name, e))
        return e

    mark("start")
    if mode == "dstore":
        from . import mvn_potrf_panel_width
        kp = mvn_potrf_panel_width(n)
        ops.dcov(d_xy_sorted, cfg, L, n, world, rank, kp)
        mark("cov")
        info = ops.potrf_dstore(L, n, group, kp)
        if info != -1:
            raise FloatingPointError(f"Sigma not SPD at row {info}")
        mark("potrf")
        mark("bcast")
        begin, end = shard_range(cfg.N * cfg.R, rank, world)
        M, S = ops.sov_dstore(L, n, d_a, cfg, begin, end, kp, group)
        mark("sov")
        combine_prefix(M, S, group, rescale=ops.rescale)
        mark("combine")
        logp = ops.finalize(M, S, cfg.N * cfg.R)
        mark("finalize")
        return logp
    if mode == "dist":
        ops.cov(d_xy_sorted, cfg, L)
        mark("cov")
        info = ops.potrf_dist(L, n, group)
        if info != -1:
            raise FloatingPointError(f"Sigma not SPD at row {info}")
        mark("potrf")
        mark("bcast")
    else:
        if rank == 0:
            ops.cov(d_xy_sorted, cfg, L)
            mark("cov")
            info = ops.potrf(L, n)
            if info != -1:
                raise FloatingPointError(f"Sigma not SPD at row {info}")
            mark("potrf")
        else:
            mark("cov")
            mark("potrf")
        broadcast_L(L, group)
        mark("bcast")
    begin, end = shard_range(cfg.N * cfg.R, rank, world)
    M, S = ops.sov(L, n, d_a, cfg, begin, end)
    mark("sov")
    combine_prefix(M, S, group, rescale=ops.rescale)
    mark("combine")
    logp = ops.finalize(M, S, cfg.N * cfg.R)
    mark("finalize")
    return logp


def potrf_launches(n: int, world: int = 1, rank: int = 0, kp: int | None = None, nsm: int = 148) -> int:
    """Kernels launched by one factorisation with super-panels of kp columns: mvn_potrf (world 1)
    or this rank's share of potrf_distributed (panel = per column [update] + POTRF [+ TRSM]; one
    update per bulk / lookahead step; pack / unpack)."""
    nt = -(-n // TILE)
    if kp is None:
        from . import mvn_potrf_panel_width
        kp = mvn_potrf_panel_width(n)
    S = -(-nt // kp)

    def panel(sp):
        k, w = sp * kp, min(kp, nt - sp * kp)
        return sum((1 if j else 0) + 1 + (1 if nt - k - j - 1 > 0 else 0) for j in range(w))

    if world == 1:
        c = panel(0)
        for sp in range(S - 1):
            kn, wn = (sp + 1) * kp, min(kp, nt - (sp + 1) * kp)
            c += (1 if kn + wn < nt else 0) + 1 + panel(sp + 1)
        return c
    c = 0
    for sp in range(S):
        c += (panel(sp) + 1) if sp % world == rank else 1        # factor + pack, or unpack
        if sp + 1 < S:
            if (sp + 1) % world == rank:
                c += 1                                            # lookahead update
            first = owned_first(sp + 1, rank, world)
            if first == sp + 1 and (sp + 1) % world == rank:
                first += world
            c += 1 if first * kp < nt else 0
    return c


# ------------------------------------------------------------------------------------- NEXT-1
TILE = 128


def owned_first(sp: int, rank: int, world: int) -> int:
    """Smallest super-panel index >= sp owned by `rank` under the 1-D block-cyclic map s -> s mod world."""
    return sp + ((rank - sp) % world)


def potrf_dist_schedule(ops, rank: int, world: int):
    """The per-rank step loop of the distributed right-looking Cholesky, as a generator.

    Super-panels of kp = ops.kp tile columns (super-panel s = columns s*kp .. s*kp+kp-1) are owned
    by rank s mod W. The generator yields ("bcast", s, src) whenever super-panel s (packed into
    ops.panel_buf(s)) must be broadcast from rank src, and is resumed with a handle that `ops.wait`
    understands. Runners: `potrf_distributed` (torch.distributed, one generator per process) and the
    single-device emulator in the tests (W generators stepped in lockstep). The recurrence is
    mvn_potrf's (Alg. 1 l.8, built from the same two library calls); only the ownership of
    the updates is split:
      panel s    : owner(s) factors super-panel s (mvn_potrf_panel) and packs it;
      lookahead  : owner(s+1) updates super-panel s+1's columns with super-panel s and factors it
                   on the side stream, whose broadcast then overlaps the bulk update of step s;
      bulk       : every rank updates its own columns after super-panel s (minus the lookahead).
    """
    nt, kp = ops.nt, ops.kp
    S = -(-nt // kp)
    owner = lambda sp: sp % world
    col = lambda sp: sp * kp
    width = lambda sp: min(kp, nt - sp * kp)
    if rank == owner(0):
        ops.panel(0, "side")
        ops.pack(0, "side")
    h = yield ("bcast", 0, owner(0))
    for sp in range(S):
        ops.wait(h, "main")                      # super-panel sp has arrived (or was produced here)
        if rank != owner(sp):
            ops.unpack(sp, "main")
        ev = ops.record("main")                  # also orders every earlier bulk update
        if sp + 1 < S:
            ops.wait(ev, "side")
            if rank == owner(sp + 1):
                ops.update(sp, col(sp + 1), nt, width(sp + 1), "side")      # the next super-panel only
                ops.panel(sp + 1, "side")
                ops.pack(sp + 1, "side")
            h = yield ("bcast", sp + 1, owner(sp + 1))
            first = owned_first(sp + 1, rank, world)
            if first == sp + 1 and rank == owner(sp + 1):
                first += world
            ops.update(sp, col(first), kp * world, kp, "main", side_busy=(rank == owner(sp + 1)))
    ops.join()


class CudaPotrfOps:
    """libmvn building blocks for potrf_dist_schedule on one device: the bulk updates on `main`
    (default: torch's current stream), the panel chain on a high-priority side stream."""

    SIDE_SMS = 4                                 # SMs left free for the panel chain (as mvn_potrf, panel_sms())

    def __init__(self, L, n: int, main=None, kp: int | None = None):
        import torch
        from . import mvn_potrf_panel_width, panel_numel
        self.torch = torch
        self.L, self.n = L, n
        self.nt = -(-n // TILE)
        self.kp = kp or mvn_potrf_panel_width(n)
        self.dev = L.device
        self.main = main if main is not None else torch.cuda.current_stream(self.dev)
        self.side = torch.cuda.Stream(device=self.dev, priority=-1)
        self.side.wait_stream(self.main)
        m = panel_numel(n, 0, self.kp)
        self.bufs = [torch.empty(m, dtype=torch.float64, device=self.dev) for _ in range(2)]

    def _st(self, which):
        return self.main if which == "main" else self.side

    def panel_buf(self, sp: int):
        from . import panel_numel
        return self.bufs[sp & 1][:panel_numel(self.n, sp * self.kp, self.kp)]

    def panel(self, sp, on):
        from . import mvn_potrf_panel
        mvn_potrf_panel(self.L, self.n, sp * self.kp, self.kp, stream=self._st(on))

    def pack(self, sp, on):
        from . import mvn_panel_pack
        mvn_panel_pack(self.L, self.n, sp * self.kp, self.kp, self.panel_buf(sp), stream=self._st(on))

    def unpack(self, sp, on):
        from . import mvn_panel_unpack
        mvn_panel_unpack(self.panel_buf(sp), self.n, sp * self.kp, self.kp, self.L, stream=self._st(on))

    def update(self, sp, c0, cs, cb, on, side_busy=True):
        from . import mvn_potrf_update
        if c0 < self.nt:
            reserve = self.SIDE_SMS if (on == "main" and side_busy) else 0
            mvn_potrf_update(self.L, self.n, sp * self.kp, self.kp, c0, cs, cb, reserve, stream=self._st(on))

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


class CudaPotrfDistOps(CudaPotrfOps):
    """potrf_dist_schedule's building blocks on a rank's LOCAL storage (NEXT-1 distributed storage,
    include/mvn.h mvn_dtiles): `local` holds only the tile columns this rank owns (~1/W of L). The
    owner factors super-panel s in place and packs it into the broadcast buffer; every rank updates
    its own columns straight from the buffer (mvn_dpotrf_update), so `unpack` is a no-op and no rank
    ever holds the whole matrix. Same arithmetic as mvn_potrf: the gathered factor is bit-identical."""

    def __init__(self, local, n: int, world: int, rank: int, main=None, kp: int | None = None):
        import torch
        from . import dtiles, mvn_dpanel_numel, mvn_potrf_panel_width
        self.torch = torch
        self.L, self.n = local, n
        self.nt = -(-n // TILE)
        self.kp = kp or mvn_potrf_panel_width(n)
        self.world, self.rank = world, rank
        self.d = dtiles(n, world, rank, self.kp)
        self.dev = local.device
        self.main = main if main is not None else torch.cuda.current_stream(self.dev)
        self.side = torch.cuda.Stream(device=self.dev, priority=-1)
        self.side.wait_stream(self.main)
        m = mvn_dpanel_numel(n, world, rank, self.kp, 0)
        self.bufs = [torch.empty(m, dtype=torch.float64, device=self.dev) for _ in range(2)]

    def panel_buf(self, sp: int):
        from . import mvn_dpanel_numel
        return self.bufs[sp & 1][:mvn_dpanel_numel(self.n, self.world, self.rank, self.kp, sp)]

    def panel(self, sp, on):
        from . import mvn_dpotrf_panel
        mvn_dpotrf_panel(self.L, self.d, sp, stream=self._st(on))

    def pack(self, sp, on):
        from . import mvn_dpanel_pack
        mvn_dpanel_pack(self.L, self.d, sp, self.panel_buf(sp), stream=self._st(on))

    def unpack(self, sp, on):
        pass                                     # updates read the broadcast buffer directly

    def update(self, sp, c0, cs, cb, on, side_busy=True, just_one=None):
        from . import mvn_dpotrf_update
        if c0 < self.nt:
            reserve = self.SIDE_SMS if (on == "main" and side_busy) else 0
            # the 1-D schedule's two forms: the lookahead (one super-panel, cs = nt) or every owned
            # super-panel from c0 on (cs = kp * W, c0 owned); the 2-D schedule says which explicitly
            if just_one is None:
                just_one = cs >= self.nt
            mvn_dpotrf_update(self.L, self.d, sp, self.panel_buf(sp), c0 // self.kp, just_one=just_one,
                              sm_reserve=reserve, stream=self._st(on))


def potrf_distributed_local(local, n: int, group=None, kp: int | None = None) -> int:
    """potrf_distributed on distributed storage: `local` is this rank's mvn_dtiles buffer (owned
    tile columns, Sigma generated there by mvn_dcov_matern); on return it holds this rank's
    columns of L. Returns info as potrf_distributed."""
    initialized = dist.is_available() and dist.is_initialized()
    world = dist.get_world_size(group) if initialized else 1
    rank = dist.get_rank(group) if initialized else 0
    _cuda_info(local)
    return potrf_distributed(local, n, group, ops=CudaPotrfDistOps(local, n, world, rank, kp=kp))


# ------------------------------------------------------------------------------------- NEXT-1, 2-D
def potrf_2d_schedule(ops, pr: int, pc: int, P: int, Q: int):
    """The per-rank step loop of the 2-D block-cyclic right-looking Cholesky on distributed storage
    (block (I, J) of kp x kp tiles owned by rank (I mod P, J mod Q)), as a generator; the same
    recurrence as mvn_potrf (bit-identical factor). Per super-step s (process column qs = s mod Q):
      diag     : rank (s mod P, qs) factors the diagonal block and packs it (mvn_dpotrf_panel / pack);
      yield ("diag", s, owner)   -> the diagonal block reaches the ranks of process column qs;
      panel    : the ranks of column qs solve their rows below it and pack them (mvn_dpanel_trsm / pack);
      yield ("panel", s, qs)     -> every rank receives the whole super-panel (its row blocks come
                                    from ranks (I mod P, qs));
      update   : every rank updates its own trailing tiles from the buffer (mvn_dpotrf_update).
    The runner resumes the generator with a handle `ops.wait` understands."""
    S = -(-ops.nt // ops.kp)
    for s in range(S):
        ps, qs = s % P, s % Q
        if (pr, pc) == (ps, qs):
            ops.panel(s, "main")
            ops.pack(s, "main")
        h = yield ("diag", s, (ps, qs))
        ops.wait(h, "main")
        if pc == qs:
            ops.trsm(s, "main")
            ops.pack(s, "main")
        h = yield ("panel", s, qs)
        ops.wait(h, "main")
        if s + 1 < S:
            ops.update(s, (s + 1) * ops.kp, ops.kp * Q, ops.kp, "main", side_busy=False, just_one=False)
    ops.join()


class CudaPotrf2DOps(CudaPotrfDistOps):
    """potrf_2d_schedule's building blocks on a rank's 2-D distributed storage (mvn_dtiles with
    prows = P): rank = pr * Q + pc holds the blocks (I, J) with I mod P = pr, J mod Q = pc."""

    def __init__(self, local, n: int, P: int, Q: int, pr: int, pc: int, main=None, kp: int | None = None):
        super().__init__(local, n, P * Q, pr * Q + pc, main=main, kp=kp)
        from . import dtiles
        self.P, self.Q, self.pr, self.pc = P, Q, pr, pc
        self.d = dtiles(n, P * Q, pr * Q + pc, self.kp, P)

    def trsm(self, sp, on):
        from . import mvn_dpanel_trsm
        mvn_dpanel_trsm(self.L, self.d, sp, self.panel_buf(sp), stream=self._st(on))

    def row_block_range(self, sp: int, I: int):
        """Element range [a, b) of row block I (tile rows I kp .. I kp + kp - 1, >= sp kp) in the
        kPanel buffer of super-panel sp (tiles (i, k .. min(i, k+w-1)) row after row)."""
        k = sp * self.kp
        w = min(self.kp, self.nt - k)

        def off(i):
            m = i - k
            return (m * (m + 1) // 2 if m <= w else w * (w + 1) // 2 + (m - w) * w) * TILE * TILE
        lo, hi = max(I * self.kp, k), min((I + 1) * self.kp, self.nt)
        return off(lo), off(hi)


def potrf_distributed_2d(local, n: int, P: int, ops=None, kp: int | None = None) -> int:
    """The 2-D block-cyclic factorisation over the default process group (W = P x Q ranks, rank =
    pr * Q + pc) on distributed storage (`local`: this rank's mvn_dtiles buffer with prows = P,
    Sigma generated by mvn_dcov_matern). The diagonal block goes to the process column by a
    broadcast in the column's subgroup; each row block of the solved super-panel is broadcast from
    its owner (I mod P, qs) to all ranks. Returns info (-1 = SPD, else the first failing row, agreed
    by all ranks). `ops` defaults to CudaPotrf2DOps (tests pass host stand-ins)."""
    W = dist.get_world_size()
    rank = dist.get_rank()
    if W % P:
        raise ValueError(f"world size {W} is not a multiple of P = {P}")
    Q = W // P
    pr, pc = rank // Q, rank % Q
    col_groups = [dist.new_group([p * Q + q for p in range(P)]) for q in range(Q)]   # same order on every rank
    if ops is None:
        _cuda_info(local)
        ops = CudaPotrf2DOps(local, n, P, Q, pr, pc, kp=kp)
    gen = potrf_2d_schedule(ops, pr, pc, P, Q)
    req = next(gen, None)
    while req is not None:
        kind, sp = req[0], req[1]
        buf = ops.panel_buf(sp)
        if kind == "diag":
            ps, qs = req[2]
            if pc == qs:
                a, b = ops.row_block_range(sp, sp)
                dist.broadcast(buf[a:b], src=ps * Q + qs, group=col_groups[qs])
        else:
            qs = req[2]
            for I in range(sp, -(-ops.nt // ops.kp)):
                a, b = ops.row_block_range(sp, I)
                if a < b:
                    dist.broadcast(buf[a:b], src=(I % P) * Q + qs)
        try:
            req = gen.send(None)
        except StopIteration:
            req = None
    info = ops.info() if hasattr(ops, "info") else _cuda_info(local)
    big = 1 << 62
    t = torch.tensor([info if info >= 0 else big], dtype=torch.int64, device=getattr(ops, "dev", "cpu"))
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    info = int(t.item())
    return -1 if info == big else info


def potrf_distributed(L, n: int, group=None, ops=None, force_collectives: bool = False) -> int:
    """Distributed tiled Cholesky of the tile-packed Sigma in `L` (every rank holds the full buffer
    with the same Sigma); on return every rank's `L` holds all of L. Returns info (-1 = SPD, else
    the first failing 0-based row, agreed over the ranks). With one rank this is the lookahead
    schedule of mvn_potrf driven from Python; force_collectives issues the NCCL broadcasts and the
    info all_reduce even then (a one-rank communicator exercises the exact multi-GPU plumbing)."""
    initialized = dist.is_available() and dist.is_initialized()
    world = dist.get_world_size(group) if initialized else 1
    rank = dist.get_rank(group) if initialized else 0
    use_comm = initialized and (world > 1 or force_collectives or FORCE_COLLECTIVES)
    if ops is None:
        _cuda_info(L)                            # reset the device pivot flag (synchronises)
        ops = CudaPotrfOps(L, n)
    gen = potrf_dist_schedule(ops, rank, world)
    req = next(gen, None)
    while req is not None:
        _, k, src = req
        h = None
        if not use_comm:
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
    if use_comm:
        big = 1 << 62
        t = torch.tensor([info if info >= 0 else big], dtype=torch.int64, device=getattr(ops, "dev", "cpu"))
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
        info = int(t.item())
        info = -1 if info == big else info
    return info


def _cuda_info(L) -> int:
    from . import mvn_potrf_info
    return mvn_potrf_info(L.device.index, reset=True)


# ---------------------------------------------------------------------------- NEXT-1, the SOV sweep
def sov_phases(nt: int, phase_rows: int) -> list[tuple[int, int]]:
    """Consecutive tile-row ranges [b, e) of phase_rows rows covering [0, nt)."""
    phase_rows = max(int(phase_rows), 1)
    return [(b, min(b + phase_rows, nt)) for b in range(0, nt, phase_rows)]


def sov_rows_schedule(ops, nphases: int):
    """The per-rank loop of the sweep over distributed L: the pieces of phase p + 1 are broadcast
    while phase p sweeps. comm(p) issues the broadcasts of phase p (asynchronous: the NCCL stream
    waits only for the work already queued, so issuing comm(p + 1) BEFORE queueing sweep(p) lets
    the transfer overlap it); wait(h) orders the compute stream after them; assemble(p) places the
    ranks' pieces in the row slice (a copy kernel on the compute stream, so it runs after sweep(p - 1)
    has read the slice); sweep(p) runs the kernels of the phase's rows. A receive buffer is rewritten
    by comm(p + 1) only after assemble(p), queued before it, has read it."""
    h = ops.comm(0) if nphases else None
    for p in range(nphases):
        ops.wait(h)
        ops.assemble(p)
        h = ops.comm(p + 1) if p + 1 < nphases else None
        ops.sweep(p)


class CudaSovRowsOps:
    """sov_rows_schedule's building blocks on a rank's distributed storage (mvn_dtiles, 1-D or 2-D):
    rank r's tiles of rows [b, e) are one contiguous piece of its buffer (mvn_drows_offset), broadcast
    from r to every rank (this rank's own piece straight from its storage) and placed in the row
    slice by mvn_drows_unpack; mvn_sweep_rows then runs the phase."""

    def __init__(self, local, n: int, world: int, rank: int, kp: int, prows: int, phases, sweep, group=None,
                 use_comm: bool = True):
        from . import dtiles, mvn_drows_offset, tile_rows_range
        self.local, self.n, self.world, self.rank = local, n, world, rank
        self.phases, self.sw, self.group, self.use_comm = phases, sweep, group, use_comm
        nt = -(-n // 128)
        self.d = [dtiles(n, world, r, kp, prows) for r in range(world)]
        self.off = [[mvn_drows_offset(self.d[r], i) for i in range(nt + 1)] for r in range(world)]
        piece = max((self.off[r][e] - self.off[r][b] for r in range(world) for b, e in phases), default=0)
        slc = max((tile_rows_range(b, e)[1] - tile_rows_range(b, e)[0] for b, e in phases), default=0)
        dev = local.device
        self.recv = {r: torch.empty(max(piece, 1), dtype=torch.float64, device=dev) for r in range(world) if r != rank}
        self.rows = torch.empty(max(slc, 1), dtype=torch.float64, device=dev)

    def piece(self, r: int, p: int):
        b, e = self.phases[p]
        lo, hi = self.off[r][b], self.off[r][e]
        return self.local[lo:hi] if r == self.rank else self.recv[r][:hi - lo]

    def comm(self, p: int):
        if not self.use_comm:
            return None
        hs = []
        for r in range(self.world):
            buf = self.piece(r, p)
            if buf.numel() == 0:
                continue
            src = dist.get_global_rank(self.group, r) if self.group is not None else r
            hs.append(dist.broadcast(buf, src=src, group=self.group, async_op=True))
        return hs

    def wait(self, hs):
        for h in hs or ():
            h.wait()

    def slice(self, p: int):
        from . import tile_rows_range
        b, e = self.phases[p]
        lo, hi = tile_rows_range(b, e)
        return self.rows[:hi - lo]

    def assemble(self, p: int):
        from . import mvn_drows_unpack
        b, e = self.phases[p]
        out = self.slice(p)
        for r in range(self.world):
            pc = self.piece(r, p)
            if pc.numel():
                mvn_drows_unpack(self.d[r], pc, b, e, out)

    def sweep(self, p: int):
        from . import mvn_sweep_rows
        b, e = self.phases[p]
        mvn_sweep_rows(self.sw, self.slice(p), b, e)


def sov_distributed(local, n: int, d_a, N: int, R: int, seed: int, begin: int, end: int, kp: int, prows: int = 1,
                    group=None, phase_rows: int = 8, force_collectives: bool = False):
    """The SOV sweep of samples [begin, end) on this rank with L on DISTRIBUTED storage (`local`:
    this rank's mvn_dtiles buffer, e.g. after potrf_distributed_local / potrf_distributed_2d), phase
    after phase of `phase_rows` tile rows, each phase's rows gathered from all ranks over NCCL while
    the previous phase sweeps. Returns this rank's (M, S) — bitwise those of mvn_sov_prefix on the
    full L for the same range — to be combined over the ranks as usual (combine_prefix)."""
    from . import mvn_sweep_begin, mvn_sweep_end
    initialized = dist.is_available() and dist.is_initialized()
    world = dist.get_world_size(group) if initialized else 1
    rank = dist.get_rank(group) if initialized else 0
    use_comm = initialized and (world > 1 or force_collectives or FORCE_COLLECTIVES)
    nt = -(-n // 128)
    phases = sov_phases(nt, phase_rows)
    sw = mvn_sweep_begin(n, d_a, N, R, seed, begin, end)
    ops = CudaSovRowsOps(local, n, world, rank, kp, prows, phases, sw, group=group, use_comm=use_comm)
    sov_rows_schedule(ops, len(phases))
    return mvn_sweep_end(sw)

