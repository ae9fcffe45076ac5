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


def crd_step(d_xy_sorted: torch.Tensor, d_a: torch.Tensor, L: torch.Tensor, cfg, group=None, events=None):
    """One pass of the whole hot path (a2..a9) on this rank; returns device log P (n,).

    events: optional list to which (name, start_event, end_event) are appended for stage timing.
    """
    from . import mvn_cov_matern, mvn_potrf, mvn_sov_prefix, mvn_prefix_finalize
    n = d_a.numel()
    world = dist.get_world_size(group) if (dist.is_available() and dist.is_initialized()) else 1
    rank = dist.get_rank(group) if world > 1 else 0

    def mark(name):
        if events is None:
            return None
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        events.append((name, e))
        return e

    mark("start")
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
