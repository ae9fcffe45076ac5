#!/usr/bin/env python
"""bench.py — one JSON line for the driver (contract in the task statement).

A step is one pass of the whole hot path on one workload:
  Matérn tiles -> tiled DMMA Cholesky -> (N>1: broadcast L) -> SOV/QMC prefix sweep over this
  rank's samples -> (N>1: allreduce combine) -> log P_k -> confidence regions (host).
Inputs (sorted locations, limits) are resident in HBM when the timed region starts; the e2e number
times the public C-ABI call mvn_crd with host buffers (H2D and D2H inside).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config D] [--impl ours|reference]

metric: BASELINE.json's "SOV-QMC n·N sample-dims/s" (value = n*N*R / step time, whole job), with
the other two BASELINE metrics (Cholesky fp64 TFLOP/s, end-to-end region time) as extra keys.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

PEAK_FP64_TFLOPS = 37.07          # measured DMMA peak on this pool (profiles/r01_fp64_calibration.md)
INT8_PEAK_POPS = 4.75             # tcgen05 kind::i8 dense, measured 8,174 MAC/clk/SM at 1,965 MHz (tools/umma_i8_test.cu)
METRIC = "SOV-QMC n·N sample-dims/s"
UNIT = "sample-dims/s"


def committed_traffic(cfg_name: str, kernel: str):
    """DRAM bytes per launch of `kernel` at this config from the committed ncu capture
    (profiles/traffic.json), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f).get(cfg_name)
        return float(t["bytes"]) if t and t.get("kernel") == kernel else None
    except (OSError, ValueError, KeyError):
        return None


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


# --------------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (SM clock, throttle reasons)."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.active",
              "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if len(r) >= 8 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 8 and r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            if len(r) < 8:
                continue
            for nm, v in zip(names, r[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------------- oracle (CPU)
def oracle_sample(cfg, n_sub: int, J: int, threads: int):
    """The oracle on a bounded sample of the workload: the leading n_sub sorted locations (the first
    n_sub prefixes are exactly the first n_sub rows of the full sweep, reading R1) with J samples of
    shift 0. Returns (seconds, details) and the full-workload time extrapolated by operation count:
    Cholesky (n/n_sub)^3, SOV (n/n_sub)^2 * NR/J."""
    import oracle
    inp = W.make_inputs(cfg)
    var = np.full(cfg.n, cfg.sigma2 + cfg.nugget)
    order, a, _ = oracle.marginal_order(inp.mu, var, cfg.u)
    sel = order[:n_sub]
    t0 = time.perf_counter()
    S = oracle.covariance(inp.xy[sel], cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget)
    t1 = time.perf_counter()
    L, info = oracle.cholesky(S, nthreads=threads)
    t2 = time.perf_counter()
    G = oracle.generators(n_sub)
    D = oracle.shifts(cfg.seed_lattice, 1, n_sub)
    chunk = max(1, -(-J // threads))
    parts = oracle.sov_units(L, a[:n_sub], np.full(n_sub, np.inf), G, D, J, 1, chunk, nthreads=threads)
    M, Ssum = oracle.combine_units(parts)
    oracle.prefix_logp(M, Ssum, J)
    t3 = time.perf_counter()
    n, NR = cfg.n, cfg.NR
    t_full = (t1 - t0) * (n / n_sub) ** 2 + (t2 - t1) * (n / n_sub) ** 3 + (t3 - t2) * (n / n_sub) ** 2 * (NR / J)
    return t3 - t0, t_full, {"cov_s": t1 - t0, "chol_s": t2 - t1, "sov_s": t3 - t2}


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def oracle_plan(cfg):
    """(n_sub, J) so that one oracle sample is ~10-20 s on ~16 cores."""
    n_sub = min(cfg.n, 8192)
    J = min(cfg.NR, 4096)
    return n_sub, J


def config_dict(cfg, world: int, mode: str) -> dict:
    """The `config` object of the JSON line; identical for both arms (ours and --impl reference)."""
    return {"workload": f"config {cfg.name}: n={cfg.n} ({cfg.g}x{cfg.g} jittered grid), Matern "
                        f"(s2={cfg.sigma2}, beta={cfg.beta}, nu={cfg.nu}) + nugget {cfg.nugget}, u={cfg.u}, "
                        f"N={cfg.N} x R={cfg.R} QMC", "n": cfg.n, "N": cfg.N, "R": cfg.R,
            "parallelism": (f"samples sharded over {world} GPU(s); " +
                            ("tiles on distributed storage (1-D block-cyclic, ~1/W per GPU), distributed "
                             "Cholesky, sweep gathering each phase's rows (NEXT-1)" if mode == "dstore"
                             else "Cholesky 1-D block-cyclic over the GPUs (NEXT-1)" if mode == "dist" and world > 1
                             else "Cholesky on rank 0, L broadcast" if world > 1 else "one GPU")),
            "l2": "flushed between timed steps (256 MB write); L itself is "
                  f"{8 * cfg.n * (cfg.n + 1) / 2 / 1e9:.2f} GB (> 126 MB L2)"}


def potrf_mode(args, world: int, force: bool) -> str:
    """--potrf auto = the north_star layout (rank 0 factors, L broadcast); dist = NEXT-1."""
    return "rank0" if args.potrf == "auto" else args.potrf


# --------------------------------------------------------------------------------- reference arm
def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    thr = cpu_threads()
    n_sub, J = oracle_plan(cfg)
    for _ in range(args.warmup):
        oracle_sample(cfg, min(n_sub, 256), min(J, 256), thr)
    times, fulls = [], []
    for _ in range(args.steps):
        t, tf, det = oracle_sample(cfg, n_sub, J, thr)
        times.append(t)
        fulls.append(tf)
    t_full = float(np.mean(fulls))
    value = cfg.n * cfg.NR / t_full
    sample = (f"oracle (oracle/, C -O2 + numpy) on the leading {n_sub} of {cfg.n} sorted locations x {J} samples "
              f"of shift 0 per step; full-workload time extrapolated by op count (Cholesky x(n/n')^3, SOV x(n/n')^2*NR/J)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_full * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(cfg, args.gpus, potrf_mode(args, args.gpus, args.force_dist)),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": thr, "kind": "oracle", "sample": sample,
                             "measured_s_per_step": float(np.mean(times))},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------------- NEXT-2 workload
def mc_chunks(n: int, draws: int) -> int:
    """Chunks mvn_mc_validate splits `draws` into (as many 128-draw blocks as fit 8 GiB of Z)."""
    n_pad = -(-n // 128) * 128
    blocks = max(1, (8 << 30) // (n_pad * 132 * 8))
    return -(-draws // (blocks * 128))


def run_mc(args, cfg):
    """MC validation of the regions on one workload: untimed cov + potrf + one CRD sweep for
    the regions k*, then K timed passes of mvn_mc_validate over --mc-samples draws (sharded over
    the ranks, counts all_reduce'd). Prints one JSON line (not the driver's headline)."""
    import torch
    import torch.distributed as dist
    import paper_2405_14892_b200 as mvn
    from paper_2405_14892_b200 import parallel

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")    # stdout: the one JSON line
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    inp = W.make_inputs(cfg)
    n = cfg.n
    var = np.full(n, cfg.sigma2 + cfg.nugget)
    order, a, _ = mvn.mvn_marginal_order(inp.mu, var, cfg.u)
    d_xy = torch.from_numpy(np.ascontiguousarray(inp.xy[order])).cuda()
    d_a = torch.from_numpy(a).cuda()
    L = mvn.alloc_tiles(n)
    logp = parallel.crd_step(d_xy, d_a, L, cfg, potrf=args.potrf)      # untimed: L and the regions
    k_star, _ = mvn.mvn_confidence_region(logp.cpu().numpy(), cfg.conf)
    Ns = args.mc_samples
    b, e = parallel.shard_range(Ns, rank, world)
    count = torch.zeros(n + 1, dtype=torch.uint64, device="cuda")
    for _ in range(args.warmup):
        count.zero_()
        mvn.mvn_mc_validate(L, n, d_a, 777, b, e, count=count, method=args.mc_method)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    if world > 1:
        dist.barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ms = []
    for _ in range(args.steps):
        count.zero_()
        ev0.record()
        mvn.mvn_mc_validate(L, n, d_a, 777, b, e, count=count, method=args.mc_method)
        ev1.record()
        torch.cuda.synchronize()
        ms.append(ev0.elapsed_time(ev1))
    clk = clocks.stop()
    t = float(np.sum(ms))
    if world > 1:
        c64 = count.to(torch.int64)
        dist.all_reduce(c64)
        count = c64
        tt = torch.tensor([t], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    ms_step = t / args.steps
    p_hat = mvn.mvn_mc_levels(count.cpu().numpy().astype(np.uint64), Ns, k_star)
    flops = float(n) * (n + 1) * (e - b)
    achieved = flops / (ms_step / 1e3) / 1e12
    line = {"metric": "MC validation draw-dims/s (NEXT-2)", "value": n * Ns / (ms_step / 1e3), "unit": "draw-dims/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"config {cfg.name}: MC validation, {Ns} draws of mu + L z", "n": n, "draws": Ns},
            "roofline": ({"kernel": "k_mc_trmm (X = L Z on DMMA + first-failure epilogue)", "bound": "tensor",
                          "achieved": achieved, "peak": PEAK_FP64_TFLOPS, "unit": "TFLOP/s",
                          "frac": achieved / PEAK_FP64_TFLOPS, "traffic": None,
                          "algorithmic": f"n(n+1) flops per draw x {e - b} draws"} if args.mc_method == 0 else
                         {"kernel": ("k_oz_trmm (X = L Z as 36 exact int8 GEMMs per 32-K chunk on tcgen05, TMEM)"
                                     if args.mc_method == 1 else
                                     "k_oz2_trmm (36 exact int8 GEMMs per 32-K chunk split by level over a 2-CTA cluster, M128 N128)"),
                          "bound": "tensor", "achieved": achieved * 36 / 1e3, "peak": INT8_PEAK_POPS, "unit": "POP/s (int8 MAC x2)",
                          "frac": achieved * 36 / 1e3 / INT8_PEAK_POPS, "traffic": None,
                          "fp64_equivalent_tflops": achieved,
                          "algorithmic": f"n(n+1) fp64-equivalent flops per draw x {e - b} draws; 36 int8 products each"}),
            "mc_method": args.mc_method,
            "levels": [float(c) for c in cfg.conf], "k_star": [int(k) for k in k_star],
            "p_hat": [float(p) for p in p_hat],
            "one_minus_alpha_minus_p_hat": [float(c - p) for c, p in zip(cfg.conf, p_hat)],
            "mc_se": [float(math.sqrt(max(p * (1 - p), 0.0) / Ns)) for p in p_hat],
            "clocks": clk, "gpu_launches": 4 * args.steps * mc_chunks(n, e - b)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


# --------------------------------------------------------------------------------- NEXT-4 / NEXT-1 workloads
def run_posterior(args):
    """Posterior conditioning (Eq. 7-8) at the paper's synthetic size: n = 40,000 sites
    (200 x 200 jittered grid, config-B kernel), m = 6,250 noisy observations (tau = 0.5). Timed:
    mvn_posterior (augmented Matérn, partial DMMA Cholesky, extraction) + marginal order +
    mvn_posterior_tiles (permutation into sorted order). Algorithmic flops: m^3/3 + m^2 n + n^2 m."""
    import torch
    import paper_2405_14892_b200 as mvn
    torch.cuda.set_device(0)
    cfg = W.small_config("posterior-40K", 200, 10_000, 8, base="B")
    m = 6_250
    P = W.make_posterior_inputs(cfg, m)
    n = cfg.n
    out = mvn.alloc_tiles(n)

    def once():
        mp, vp = mvn.mvn_posterior(P.xy, P.mu, P.obs, P.y, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget, P.tau)
        order, a, _ = mvn.mvn_marginal_order(mp, vp, cfg.u)
        mvn.mvn_posterior_tiles(order, out=out)
        return order

    for _ in range(max(1, args.warmup)):
        once()
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        once()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    t = float(np.mean(ts))
    mp_ = -(-m // 128) * 128
    flops = mp_ ** 3 / 3 + mp_ ** 2 * n + float(n) ** 2 * mp_
    line = {"metric": "posterior conditioning time (NEXT-4)", "value": t * 1e3, "unit": "ms", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": False,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{n} sites (200x200 jittered grid, Matern s2=1, beta=0.1, nu=0.5), "
                                   f"{m} observations, tau=0.5 (P:369)", "n": n, "m": m},
            "roofline": {"bound": "tensor", "achieved": flops / t / 1e12, "peak": PEAK_FP64_TFLOPS, "unit": "TFLOP/s",
                         "frac": flops / t / 1e12 / PEAK_FP64_TFLOPS,
                         "algorithmic": "m^3/3 + m^2 n + n^2 m (C factor, TRSM, SYRK of the Schur complement); "
                                        "host-timed incl. H2D/D2H of n-vectors and the permutation"}}
    print(json.dumps(line), flush=True)
    return 0


def run_potrf_dist(args, cfg):
    """NEXT-1 on one GPU: the distributed schedule (parallel.potrf_distributed, W = 1, one generator
    driven from Python, one ABI call per building block) against mvn_potrf (the same kernels driven
    from C++): the cost of the Python step loop and of the generic schedule."""
    import torch
    import paper_2405_14892_b200 as mvn
    from paper_2405_14892_b200 import parallel
    torch.cuda.set_device(0)
    inp = W.make_inputs(cfg)
    n = cfg.n
    order, a, _ = mvn.mvn_marginal_order(inp.mu, np.full(n, cfg.sigma2 + cfg.nugget), cfg.u)
    d_xy = torch.from_numpy(np.ascontiguousarray(inp.xy[order])).cuda()
    L = mvn.alloc_tiles(n)
    res = {}
    for name, fn in [("mvn_potrf", lambda: mvn.mvn_potrf(L, n)), ("potrf_distributed_w1", lambda: parallel.potrf_distributed(L, n))]:
        ts = []
        for it in range(args.steps + 1):
            mvn.mvn_cov_matern(d_xy, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget, out=L)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            assert fn() == -1
            e1.record()
            torch.cuda.synchronize()
            if it:
                ts.append(e0.elapsed_time(e1))
        res[name] = float(np.mean(ts))
    flops = n ** 3 / 3
    line = {"metric": "Cholesky fp64 TFLOP/s, distributed schedule at W = 1 (NEXT-1)",
            "value": flops / (res["potrf_distributed_w1"] / 1e3) / 1e12, "unit": "TFLOP/s", "n_gpus": 1,
            "steps": args.steps, "higher_is_better": True, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"config {cfg.name}: n={n}", "n": n,
                       "kp": mvn.mvn_potrf_panel_width(n)},
            "ms": res, "mvn_potrf_tflops": flops / (res["mvn_potrf"] / 1e3) / 1e12,
            "launches_per_rank_w8": [parallel.potrf_launches(n, 8, r) for r in range(8)]}
    print(json.dumps(line), flush=True)
    return 0


def run_potrf_share(args, cfg):
    """NEXT-1 per-rank share on one GPU: rank 0's own work in the distributed Cholesky at W ranks
    (parallel.potrf_dist_schedule: its panels, lookahead and bulk updates of its tile columns), with
    every other rank's broadcast replaced by a local pack of that super-panel from the finished
    factor (what the NCCL receive would deliver; the network time itself, which the schedule
    overlaps with the bulk update, is not included). Checks that rank 0's columns come out bitwise
    equal to mvn_potrf's, and reports the time against mvn_potrf at W = 1: an estimate of the
    Cholesky's per-rank time at W GPUs (max over ranks ~ rank 0: it owns super-panel 0, the
    heaviest)."""
    import torch
    import paper_2405_14892_b200 as mvn
    from paper_2405_14892_b200 import parallel
    torch.cuda.set_device(0)
    inp = W.make_inputs(cfg)
    n = cfg.n
    order, a, _ = mvn.mvn_marginal_order(inp.mu, np.full(n, cfg.sigma2 + cfg.nugget), cfg.u)
    d_xy = torch.from_numpy(np.ascontiguousarray(inp.xy[order])).cuda()
    Lref = mvn.mvn_cov_matern(d_xy, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    assert mvn.mvn_potrf(Lref, n) == -1
    e1.record()
    torch.cuda.synchronize()
    full_ms = e0.elapsed_time(e1)
    kp = mvn.mvn_potrf_panel_width(n)
    nt = -(-n // 128)
    L = mvn.alloc_tiles(n)
    shares = {}
    for w in [int(x) for x in args.shard.split(",")]:
        ts, exact = [], None
        for it in range(args.steps + 1):
            mvn.mvn_cov_matern(d_xy, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget, out=L)
            torch.cuda.synchronize()
            ops = parallel.CudaPotrfOps(L, n)
            gen = parallel.potrf_dist_schedule(ops, 0, w)
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(ops.main)
            ops.side.wait_stream(ops.main)
            req = next(gen)
            while True:
                _, k, src = req
                if src != 0:                      # the panel another rank would broadcast
                    with torch.cuda.stream(ops.side):
                        mvn.mvn_panel_pack(Lref, n, k * kp, kp, ops.panel_buf(k), stream=ops.side)
                h = ops.record("side")
                try:
                    req = gen.send(h)
                except StopIteration:
                    break
            ops.main.wait_stream(ops.side)
            s1.record(ops.main)
            torch.cuda.synchronize()
            if it:
                ts.append(s0.elapsed_time(s1))
        # rank 0's super-panels (0, w, 2w, ...) against the single-GPU factor, bitwise
        Lh, Rh = L.view(-1), Lref.view(-1)
        same = True
        for sp in range(0, -(-nt // kp), w):
            for j in range(sp * kp, min(nt, sp * kp + kp)):
                for i in range(j, nt):
                    off = ((i * (i + 1)) // 2 + j) * 128 * 128
                    if i == j or (i - j) % 37 == 0:     # a sample of the column's tiles
                        same &= bool(torch.equal(Lh[off:off + 128 * 128], Rh[off:off + 128 * 128]))
        exact = same
        ms = float(np.mean(ts))
        shares[str(w)] = {"rank0_ms": ms, "vs_full": ms / full_ms, "ideal": 1.0 / w,
                          "rank0_columns_bitwise_equal_sampled": exact}
    line = {"metric": "distributed Cholesky: rank 0's per-rank time at W GPUs (NEXT-1, compute share)", "unit": "ms",
            "value": shares[str(max(int(x) for x in args.shard.split(",")))]["rank0_ms"], "higher_is_better": False,
            "n_gpus": 1, "steps": args.steps, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"config {cfg.name}: n={n}, rank 0's schedule with the other ranks' panels "
                                   f"delivered by local copies", "n": n, "kp": kp},
            "mvn_potrf_ms": full_ms, "shares": shares}
    print(json.dumps(line), flush=True)
    return 0


def run_shard(args, cfg):
    """Per-rank shard efficiency on one GPU: the SOV sweep (k_sov + k_reduce_blocks, through
    mvn_sov_prefix) over rank 0's 1/W share of the config's N*R samples, the exact range rank 0
    sweeps at W GPUs (parallel.shard_range), for each W in --shard. Cov + Cholesky untimed; each
    range timed --steps times with CUDA events after --warmup sweeps. Roofline: n(n-1) flops per
    sample against the fp64 DMMA peak."""
    import torch
    import paper_2405_14892_b200 as mvn
    from paper_2405_14892_b200 import parallel
    torch.cuda.set_device(0)
    inp = W.make_inputs(cfg)
    n, NR = cfg.n, cfg.NR
    order, a, _ = mvn.mvn_marginal_order(inp.mu, np.full(n, cfg.sigma2 + cfg.nugget), cfg.u)
    d_xy = torch.from_numpy(np.ascontiguousarray(inp.xy[order])).cuda()
    d_a = torch.from_numpy(a).cuda()
    L = mvn.mvn_cov_matern(d_xy, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget)
    assert mvn.mvn_potrf(L, n) == -1
    shards = {}
    clocks = ClockSampler(0)
    clocks.start()
    for w in [int(x) for x in args.shard.split(",")]:
        b, e = parallel.shard_range(NR, 0, w)
        for _ in range(args.warmup):
            mvn.mvn_sov_prefix(L, n, d_a, cfg.N, cfg.R, cfg.seed_lattice, b, e)
        ts = []
        for _ in range(args.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            mvn.mvn_sov_prefix(L, n, d_a, cfg.N, cfg.R, cfg.seed_lattice, b, e)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = float(np.mean(ts))
        per_cta = (e - b) / min(e - b, 148)
        tf = float(n) * (n - 1) * (e - b) / (ms / 1e3) / 1e12
        cnt = math.ceil(per_cta)                             # the largest CTA share (k_sov block_geom)
        nblk, units = -(-cnt // 128), -(-cnt // 8)
        shards[str(w)] = {"samples": e - b, "samples_per_cta": per_cta, "blocks_per_cta": nblk,
                          "widest_block": 8 * -(-units // nblk), "padding": 8 * units / cnt - 1,
                          "sov_ms": ms, "tflops": tf, "frac": tf / PEAK_FP64_TFLOPS, "ms_each": ts}
    clk = clocks.stop()
    line = {"metric": "SOV per-rank shard efficiency (fraction of the fp64 DMMA peak)", "unit": "frac",
            "value": min(v["frac"] for v in shards.values()), "higher_is_better": True, "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"config {cfg.name}: rank 0's share of N*R = {NR} samples at W GPUs", "n": n,
                       "N": cfg.N, "R": cfg.R},
            "shards": shards, "peak": PEAK_FP64_TFLOPS, "clocks": clk}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------------- NEXT-3 workload
def run_tlr(args):
    """TLR compression (NEXT-3 part, R23) at the paper's accuracy setting: n = 40,000 sites
    (200 x 200 jittered grid), exponential kernel, sigma^2 = 1, beta = 0.1 (medium correlation),
    Sigma in the sorted order, eps = --tlr-eps. Timed on the device (CUDA events around
    mvn_tlr_compress on its stream): the compression of all 48,828 off-diagonal tiles; the copy of the
    dense Sigma into the working buffer before each step is outside the events. Algorithmic flops
    per tile: 12 nb^3 (the Golub-Van Loan count of an nb x nb SVD with Sigma and V) + 4 nb^2 k (the
    projection A V_k V_k^T), nb = 128."""
    import torch
    import paper_2405_14892_b200 as mvn
    torch.cuda.set_device(0)
    cfg = W.small_config("tlr-40K", 200, 10_000, 8, base="B")
    inp = W.make_inputs(cfg)
    n = cfg.n
    order, a, _ = mvn.mvn_marginal_order(inp.mu, np.full(n, cfg.sigma2 + cfg.nugget), cfg.u)
    d_xs = torch.from_numpy(np.ascontiguousarray(inp.xy[order])).cuda()
    base = mvn.mvn_cov_matern(d_xs, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget)
    T = torch.empty_like(base)
    nt = -(-n // 128)
    ntiles = nt * (nt - 1) // 2
    ranks = torch.empty(ntiles, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream()
    ts = []
    for it in range(args.warmup + args.steps):
        T.copy_(base)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        mvn.mvn_tlr_compress(T, n, args.tlr_eps, ranks, mode=args.tlr_mode)
        e1.record(st)
        torch.cuda.synchronize()
        if it >= args.warmup:
            ts.append(e0.elapsed_time(e1))
    ms = float(np.mean(ts))
    r = ranks.cpu().numpy()
    flops = ntiles * 12.0 * 128 ** 3 + 4.0 * 128 ** 2 * float(r.sum())
    achieved = flops / (ms / 1e3) / 1e12
    info = mvn.mvn_potrf(T, n, raise_on_numeric=False)
    line = {"metric": "TLR compression time (NEXT-3)", "value": ms, "unit": "ms", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{n} sites (200x200 jittered grid, exponential kernel s2=1, beta=0.1), sorted order, "
                                   f"128-wide tiles, eps={args.tlr_eps:g} (P:368, P:439)", "n": n, "tiles": ntiles,
                       "eps": args.tlr_eps, "mode": args.tlr_mode},
            "roofline": {"bound": "alu", "achieved": achieved, "peak": PEAK_FP64_TFLOPS, "unit": "TFLOP/s",
                         "frac": achieved / PEAK_FP64_TFLOPS, "traffic": None,
                         "algorithmic": "12 nb^3 (SVD with Sigma and V, Golub-Van Loan) + 4 nb^2 k per tile; peak = the "
                                        "fp64 pipe (64 FMA/clk/SM x 148 x 1.965 GHz = 37.2 TF nominal, shared with DMMA, "
                                        "measured 37.07)"},
            "ranks": {"mean": float(r.mean()), "p90": float(np.percentile(r, 90)), "max": int(r.max())},
            "potrf_info_after": int(info), "gpu_launches": args.steps}
    print(json.dumps(line), flush=True)
    return 0


def tlr_update_flops(ranks: np.ndarray, nt: int) -> float:
    """Algorithmic flops of the factored updates of the TLR Cholesky (R26): per (i, j, k), k < j <= i,
    4 nb r_ik r_jk (M = V_ik^T V_jk, Z = U_ik M) + 2 nb^2 r_jk (T_i -= Z U_jk^T), nb = 128."""
    r = np.zeros((nt, nt))
    for I in range(1, nt):
        r[I, :I] = ranks[I * (I - 1) // 2:I * (I - 1) // 2 + I]
    tot = 0.0
    for j in range(1, nt):
        rj = r[j, :j]                                  # r_jk, k < j
        ri = r[j:, :j].copy()                          # r_ik, i >= j (row j itself: r_jk)
        tot += 4.0 * 128 * float((ri * rj).sum()) + 2.0 * 128 ** 2 * float(rj.sum()) * (nt - j)
    return tot


def run_tlr_potrf(args):
    """NEXT-3: the TLR Cholesky (mvn_tlr_potrf, R26) against the dense DMMA Cholesky (mvn_potrf) on the
    same matrix: the paper's accuracy setting — n = 40,000 sites (200 x 200 jittered grid),
    exponential kernel, sigma^2 = 1, beta = 0.1 — at eps = --tlr-eps, in the order Alg. 1 factors
    (sorted by marginal probability, R1) or in the grid's own order (--tlr-order spatial: the setting
    of the paper's rank figure, where tiles are low rank). Both timed on the device with
    CUDA events (Sigma copied into the working buffer outside the events; the TLR time includes the
    compression of Sigma). value = TLR time; roofline = the factored-update flops (tlr_update_flops)
    over the TLR time against the fp64 DMMA peak."""
    import torch
    import paper_2405_14892_b200 as mvn
    torch.cuda.set_device(0)
    cfg = W.small_config("tlr-40K", args.tlr_g, 10_000, 8, base="B")
    inp = W.make_inputs(cfg)
    n = cfg.n
    if args.tlr_order == "sorted":
        order, a, _ = mvn.mvn_marginal_order(inp.mu, np.full(n, cfg.sigma2 + cfg.nugget), cfg.u)
    else:
        order = np.arange(n)
    d_xs = torch.from_numpy(np.ascontiguousarray(inp.xy[order])).cuda()
    base = mvn.mvn_cov_matern(d_xs, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget)
    T = torch.empty_like(base)
    nt = -(-n // 128)
    noff = nt * (nt - 1) // 2
    U = torch.empty((noff, args.tlr_kmax, 128), dtype=torch.float64, device="cuda")
    V = torch.empty_like(U)
    st = torch.cuda.current_stream()

    def timed(fn):
        ts = []
        for it in range(args.warmup + args.steps):
            T.copy_(base)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            out = fn()
            e1.record(st)
            torch.cuda.synchronize()
            if it >= args.warmup:
                ts.append(e0.elapsed_time(e1))
        return float(np.mean(ts)), out

    clocks = ClockSampler(0)
    clocks.start()
    ms_tlr, f = timed(lambda: mvn.mvn_tlr_potrf(T, n, args.tlr_eps, mode=args.tlr_mode, kmax=args.tlr_kmax, U=U, V=V))
    ms_dense, info_d = timed(lambda: mvn.mvn_potrf(T, n, raise_on_numeric=False))
    # the SOV sweep on L~: dense (k_sov on the reconstructed tiles) vs the factored update
    # (k_sov_tlr), the same samples; T holds the last dense factor, so refactor with TLR first
    T.copy_(base)
    f = mvn.mvn_tlr_potrf(T, n, args.tlr_eps, mode=args.tlr_mode, kmax=args.tlr_kmax, U=U, V=V)
    a_ord = np.ascontiguousarray(cfg.u - inp.mu[order])
    d_a = torch.from_numpy(a_ord).cuda()
    ns = args.tlr_sov_samples
    sov = {}
    for name, fn in [("dense", lambda: mvn.mvn_sov_prefix(T, n, d_a, cfg.N, cfg.R, cfg.seed_lattice, 0, ns)),
                     ("factored", lambda: mvn.mvn_sov_prefix_tlr(T, f, n, d_a, cfg.N, cfg.R, cfg.seed_lattice, 0, ns))]:
        ts = []
        for it in range(args.warmup + args.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            M_, S_ = fn()
            e1.record(st)
            torch.cuda.synchronize()
            if it >= args.warmup:
                ts.append(e0.elapsed_time(e1))
        lp = (M_ + torch.log(S_) - math.log(ns)).cpu().numpy()
        sov[name] = {"ms": float(np.mean(ts)), "logp": lp}
    clk = clocks.stop()
    rL, rS = f.ranks.cpu().numpy(), f.ranks_sigma.cpu().numpy()
    flops = tlr_update_flops(rL, nt)
    achieved = flops / (ms_tlr / 1e3) / 1e12
    dense_flops = float(n) ** 3 / 3
    line = {"metric": "TLR Cholesky time (NEXT-3)", "value": ms_tlr, "unit": "ms", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_tlr, "higher_is_better": False,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{n} sites ({args.tlr_g}x{args.tlr_g} jittered grid, exponential kernel s2=1, "
                                   f"beta=0.1), {args.tlr_order} order, 128-wide tiles, eps={args.tlr_eps:g} "
                                   f"(P:368, P:439)", "n": n, "order": args.tlr_order, "eps": args.tlr_eps,
                       "mode": args.tlr_mode, "kmax": args.tlr_kmax},
            "dense_potrf_ms": ms_dense, "dense_tflops": dense_flops / (ms_dense / 1e3) / 1e12,
            "tlr_over_dense": ms_tlr / ms_dense, "info": f.info, "dense_info": int(info_d),
            "ranks_L": {"mean": float(rL.mean()), "p90": float(np.percentile(rL, 90)), "max": int(rL.max())},
            "ranks_sigma": {"mean": float(rS.mean()), "max": int(rS.max())},
            "update_flops": flops, "update_flops_over_dense_potrf": flops / dense_flops,
            "sov_on_Ltilde": {"samples": ns, "dense_ms": sov["dense"]["ms"], "factored_ms": sov["factored"]["ms"],
                              "max_abs_dlogP": float(np.max(np.abs(sov["dense"]["logp"] - sov["factored"]["logp"])))},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": PEAK_FP64_TFLOPS, "unit": "TFLOP/s",
                         "frac": achieved / PEAK_FP64_TFLOPS, "traffic": None,
                         "algorithmic": "factored updates 4 nb r_ik r_jk + 2 nb^2 r_jk per (i, j, k) over the TLR "
                                        "time (compressions and panels count as overhead)"},
            "clocks": clk, "gpu_launches": tlr_potrf_launches(nt) * args.steps}
    print(json.dumps(line), flush=True)
    return 0


def tlr_potrf_launches(nt: int) -> int:
    """Kernels mvn_tlr_potrf launches (mvn_api.cu / kernels_tlr.cu launch_tlr_potrf): the compression
    of Sigma (one launch per column), per column j the expansion, 3 per chunk of k (M, Z, accumulate), K2, K3 and the
    compression of the column, and the final expansion."""
    need = max(1, (nt // 2) * ((nt + 1) // 2))
    chunk = max(min(need, 2048), nt)
    cnt = (nt - 1) + 1 if nt > 1 else 0                   # Sigma's columns, the final expansion
    def chunks(ka, kb, rows):
        c = 0
        kc = max(1, min(kb - ka, chunk // rows))
        for k0 in range(ka, kb, kc):
            kcc = min(kc, kb - k0)
            nsplit = min(kcc, max(1, (2 * 148 + 4 * rows - 1) // (4 * rows)))
            c += 3 + (1 if nsplit > 1 else 0)
        return c
    for j in range(nt):
        rows = nt - j
        if j >= 2:
            cnt += chunks(0, j - 1, rows)                 # the columns k < j - 1 (overlapping the compression of j - 1)
        if j >= 1:
            cnt += chunks(j - 1, j, rows)                 # k = j - 1, after it
        cnt += 1 + (3 if rows > 1 else 0)
    return cnt


# --------------------------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="D", choices=sorted(W.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-shift-se", action="store_true",
                    help="skip the untimed per-shift sweeps that give the QMC standard error (qmc_error)")
    ap.add_argument("--potrf", default="auto", choices=["auto", "rank0", "dist", "dstore"],
                    help="N>1: factor on rank 0 + broadcast L (north_star), or distributed (NEXT-1); "
                         "dstore: NEXT-1 on distributed storage end to end (each rank holds ~1/N of the "
                         "tiles; the sweep gathers each phase's rows, --phase-rows); auto = rank0")
    ap.add_argument("--phase-rows", type=int, default=16,
                    help="--potrf dstore: tile rows per phase of the sweep over distributed L")
    ap.add_argument("--force-dist", action="store_true",
                    help="testing: run the multi-GPU code path (NCCL process group, distributed Cholesky, "
                         "all_reduce combine, pinned-buffer e2e) even with one rank")
    ap.add_argument("--sov-method", type=int, default=0, choices=[0, 1],
                    help="crd: 0 = SOV GEMM on fp64 DMMA (default, the headline); 1 = on the int8 tensor cores "
                         "(NEXT-4 mixed precision, Ozaki split, reading R24) - its own bench line")
    ap.add_argument("--potrf-method", type=int, default=0, choices=[0, 1, 2],
                    help="crd: 0 = Cholesky updates on fp64 DMMA (default); 1 = on the int8 tensor cores (NEXT-4, R25); "
                         "2 = the TLR Cholesky at --tlr-eps (NEXT-3, R26)")
    ap.add_argument("--shard", default="1,2,4,8", help="--workload shard: the world sizes W whose rank-0 share is timed")
    ap.add_argument("--workload", default="crd", choices=["crd", "mc", "posterior", "potrf-dist", "potrf-share", "tlr", "tlr-potrf", "shard"],
                    help="crd: the hot path (default, the driver's line); mc: NEXT-2 MC validation of the regions; "
                         "posterior: NEXT-4 conditioning (paper size: 200x200 sites, 6,250 observations); "
                         "potrf-dist: NEXT-1 schedule driven from Python vs mvn_potrf on one GPU; "
                         "tlr: NEXT-3 TLR compression at the paper's 40K-site accuracy setting; "
                         "shard: the SOV over rank 0's 1/W sample share for each W in --shard (one GPU)")
    ap.add_argument("--tlr-eps", type=float, default=1e-3, help="--workload tlr: accuracy eps (R23)")
    ap.add_argument("--tlr-order", default="sorted", choices=["sorted", "spatial"],
                    help="--workload tlr-potrf: factor Sigma in the sorted order (Alg. 1) or the grid order")
    ap.add_argument("--tlr-kmax", type=int, default=128, help="--workload tlr-potrf: factor slot width")
    ap.add_argument("--tlr-g", type=int, default=200, help="--workload tlr-potrf: grid side (n = g^2)")
    ap.add_argument("--tlr-sov-samples", type=int, default=10_000,
                    help="--workload tlr-potrf: samples of the dense vs factored SOV sweep on L~")
    ap.add_argument("--tlr-mode", type=int, default=0, choices=[0, 1],
                    help="--workload tlr: 0 = keep sigma_i >= eps, 1 = relative Frobenius error <= eps per tile")
    ap.add_argument("--mc-samples", type=int, default=50_000, help="--workload mc: draws (paper: N = 50,000, P:595)")
    ap.add_argument("--mc-method", type=int, default=0, choices=[0, 1, 2],
                    help="--workload mc: 0 = fp64 DMMA, 1 = int8 tensor cores (tcgen05 Ozaki emulation, M128 N64), "
                         "2 = the same at M128 N128 with the products split by level over a 2-CTA cluster")
    args = ap.parse_args()
    cfg = W.CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)
    if args.workload == "mc":
        return run_mc(args, cfg)
    if args.workload == "tlr":
        return run_tlr(args)
    if args.workload == "tlr-potrf":
        return run_tlr_potrf(args)
    if args.workload == "posterior":
        return run_posterior(args)
    if args.workload == "potrf-share":
        return run_potrf_share(args, cfg)
    if args.workload == "potrf-dist":
        return run_potrf_dist(args, cfg)
    if args.workload == "shard":
        return run_shard(args, cfg)

    import torch
    import torch.distributed as dist
    import paper_2405_14892_b200 as mvn
    from paper_2405_14892_b200 import parallel

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    multi = world > 1 or args.force_dist                 # the multi-GPU code path
    if multi:
        # NCCL's banner / debug lines go to stdout by default: keep stdout for the one JSON line
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 1000))
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
            parallel.FORCE_COLLECTIVES = True
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={world}"

    # ---- untimed setup: host inputs, a1 (marginal order), upload
    inp = W.make_inputs(cfg)
    n, NR = cfg.n, cfg.NR
    var = np.full(n, cfg.sigma2 + cfg.nugget)
    order, a, _ = mvn.mvn_marginal_order(inp.mu, var, cfg.u)
    d_xy = torch.from_numpy(np.ascontiguousarray(inp.xy[order])).cuda()
    d_a = torch.from_numpy(a).cuda()
    mode = potrf_mode(args, world, args.force_dist)
    if mode == "dstore":
        if (args.sov_method, args.potrf_method) != (0, 0):
            raise SystemExit("--potrf dstore runs the fp64 path (--sov-method 0 --potrf-method 0)")
        L = mvn.alloc_dtiles(n, world, rank, mvn.mvn_potrf_panel_width(n))
    else:
        L = mvn.alloc_tiles(n)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")   # 256 MB > 126 MB L2
    step_ops = parallel.crd_ops(args.sov_method, args.potrf_method, args.tlr_eps)
    if mode == "dstore":
        step_ops = type("LibmvnCrdOpsPhases", (step_ops,), {"phase_rows": args.phase_rows})

    def step(events=None):
        logp = parallel.crd_step(d_xy, d_a, L, cfg, events=events, potrf=mode, ops=step_ops)
        lp = logp.cpu().numpy()                          # a10 on the host: regions
        k, _ = mvn.mvn_confidence_region(lp, cfg.conf)
        return lp, k

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    if multi:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms, stage = [], {}
    for _ in range(args.steps):
        flush.zero_()                                    # L2 flush between timed iterations (untimed)
        ev = []
        lp, k = step(events=ev)
        e_end = torch.cuda.Event(enable_timing=True)
        e_end.record()
        torch.cuda.synchronize()
        names = [x[0] for x in ev]
        for (nm0, e0), (nm1, e1) in zip(ev[:-1], ev[1:]):
            stage.setdefault(nm1, []).append(e0.elapsed_time(e1))
        stage.setdefault("region", []).append(ev[-1][1].elapsed_time(e_end))
        step_ms.append(ev[0][1].elapsed_time(e_end))
    torch.cuda.synchronize()
    if multi:
        dist.barrier()
    clk = clocks.stop()

    total_ms = float(np.sum(step_ms))
    if multi:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        mine = torch.tensor([np.mean(stage[k]) for k in sorted(stage)], dtype=torch.float64, device="cuda")
        every = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(every, mine)
        per_rank = torch.stack(every).cpu().numpy()              # [rank][stage]
        stage_mean = dict(zip(sorted(stage), per_rank.max(axis=0).tolist()))
        stage_per_rank = {k: per_rank[:, i].tolist() for i, k in enumerate(sorted(stage))}
    else:
        stage_mean = {k: float(np.mean(v)) for k, v in stage.items()}
        stage_per_rank = None
    ms_per_step = total_ms / args.steps
    value = n * NR / (ms_per_step / 1e3)

    # ---- e2e through the public API with host buffers. N = 1: the C-ABI call mvn_crd (a1 on the
    # host, H2D of sorted locations and limits, a2..a8, D2H of log P, a10). N > 1: the same steps
    # through parallel.crd_step on every rank from pinned host buffers, max over ranks.
    e2e = None
    if not args.no_e2e and not multi and mode != "dstore":
        ts = []
        for it in range(4):                      # one warm-up call (allocations), three timed
            t0 = time.perf_counter()
            out = mvn.mvn_crd(inp.xy, inp.mu, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget, cfg.u, cfg.N, cfg.R,
                              cfg.seed_lattice, cfg.conf,
                              method=args.sov_method | (2 if args.potrf_method == 1 else 4 if args.potrf_method == 2 else 0),
                              tlr_eps=args.tlr_eps)
            t1 = time.perf_counter()
            if it > 0:
                ts.append(t1 - t0)
        e2e = {"value": n * NR / float(np.mean(ts)), "unit": UNIT, "h2d_bytes_per_step": 24 * n,
               "d2h_bytes_per_step": 8 * n, "s_per_call": float(np.mean(ts)), "calls": len(ts),
               "s_per_call_each": [float(t) for t in ts], "api": "mvn_crd (C ABI)",
               "k_star_matches_device_path": bool(np.array_equal(out.k_star, k))}
    elif not args.no_e2e:
        import torch as _t
        h_xy = _t.empty((n, 2), dtype=_t.float64).pin_memory()
        h_a = _t.empty(n, dtype=_t.float64).pin_memory()
        h_lp = _t.empty(n, dtype=_t.float64).pin_memory()
        ts = []
        for _ in range(3):
            if multi:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            o2, a2, _ = mvn.mvn_marginal_order(inp.mu, var, cfg.u)              # a1 (host)
            h_xy.numpy()[:] = inp.xy[o2]
            h_a.numpy()[:] = a2
            d_xy.copy_(h_xy, non_blocking=True)
            d_a.copy_(h_a, non_blocking=True)
            logp = parallel.crd_step(d_xy, d_a, L, cfg, potrf=mode, ops=step_ops)
            h_lp.copy_(logp, non_blocking=True)
            torch.cuda.synchronize()
            k2, _ = mvn.mvn_confidence_region(h_lp.numpy(), cfg.conf)          # a10 (host)
            t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
            if multi:
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ts.append(float(t.item()))
        e2e = {"value": n * NR / float(np.mean(ts)), "unit": UNIT, "h2d_bytes_per_step": 24 * n,
               "d2h_bytes_per_step": 8 * n, "s_per_call": float(np.mean(ts)), "calls": len(ts),
               "api": "parallel.crd_step from pinned host buffers, max over ranks",
               "k_star_matches_device_path": bool(np.array_equal(k2, k))}

    # ---- QMC error of the estimates (untimed): the per-shift estimates log P^(r) (one sweep per
    # shift, mvn_sov_prefix_shifts) and the relative standard error across the R shifts (O6, R11)
    qmc_err = None
    if rank == 0 and world == 1 and mode != "dstore" and not args.no_shift_se:
        t0 = time.perf_counter()
        Ls = mvn.mvn_sov_prefix_shifts(L, n, d_a, cfg.N, cfg.R, cfg.seed_lattice).cpu().numpy()
        lps, rse = mvn.mvn_prefix_shift_stats(Ls)
        ks = [int(x) for x in k]
        fin = np.isfinite(lp)
        qmc_err = {"R": cfg.R, "what": "relative standard error of P_k across the R randomised lattice shifts "
                                      "(sd_r P^(r)_k / (sqrt(R) mean_r P^(r)_k), ~ the standard error of log P_k)",
                   "rel_se_at_k_star": [float(rse[x - 1]) if x > 0 else None for x in ks],
                   "max_rel_se_up_to_max_k_star": float(np.nanmax(rse[:max(ks)])) if max(ks) > 0 else None,
                   "combined_vs_step_max_abs_dlogP": float(np.max(np.abs(lps[fin] - lp[fin]))),
                   "seconds": time.perf_counter() - t0}

    # ---- roofline of the dominant kernel (k_sov, SOV GEMM + chain), from the live stage times
    sov_ms = stage_mean["sov"]
    my_begin, my_end = parallel.shard_range(NR, rank, world)
    my_samples = my_end - my_begin
    sov_flops = float(n) * (n - 1) * my_samples       # algorithmic: sum_k 2(k-1) per sample (a6 + in-block dot)
    achieved = sov_flops / (sov_ms / 1e3) / 1e12
    if args.sov_method == 1:
        # int8 work of the emulated GEMM: 36 exact products over the off-diagonal row-block part,
        # sum_{rb >= 1} 128 rows x 128 rb K per sample
        nrb = -(-n // 128)
        i8_ops = 2.0 * 36 * 128 * 128 * (nrb * (nrb - 1) / 2) * my_samples
        sov_roof = {"kernel": "k_sov_oz (SOV GEMM as 36 exact int8 tcgen05 products per K-chunk, 2-CTA level split; "
                              "fp64 Phi chain)", "bound": "tensor", "achieved": i8_ops / (sov_ms / 1e3) / 1e15,
                    "peak": INT8_PEAK_POPS, "unit": "POP/s (int8)",
                    "frac": i8_ops / (sov_ms / 1e3) / 1e15 / INT8_PEAK_POPS,
                    "traffic": committed_traffic(cfg.name + "-int8", "k_sov_oz"),
                    "fp64_equivalent_tflops": achieved, "fp64_equivalent_frac_of_dmma_peak": achieved / PEAK_FP64_TFLOPS,
                    "peak_source": "int8 tcgen05 dense, measured 8,174 MAC/clk/SM at 1,965 MHz (tools/umma_i8_test.cu)",
                    "algorithmic": f"2 x 36 x 128^2 x nrb(nrb-1)/2 int8 ops per sample x {my_samples} samples "
                                   f"(= n(n-1) fp64-equivalent flops per sample)"}
    else:
        sov_roof = {"kernel": "k_sov (SOV DMMA GEMM + Phi chain)", "bound": "tensor", "achieved": achieved,
                    "peak": PEAK_FP64_TFLOPS, "unit": "TFLOP/s", "frac": achieved / PEAK_FP64_TFLOPS,
                    "traffic": committed_traffic(cfg.name, "k_sov"),
                    "peak_source": "measured fp64 DMMA peak (tools/calib_fp64.cu, profiles/r01_fp64_calibration.md); "
                                   "MEASURED_PEAKS.json has no fp64 entry",
                    "algorithmic": f"n(n-1) flops per sample x {my_samples} samples"}
    if mode in ("dist", "dstore"):
        n_potrf = parallel.potrf_launches(n, world, rank)
    else:
        n_potrf = (parallel.potrf_launches(n) if args.potrf_method != 2 else tlr_potrf_launches(-(-n // 128))) \
            if rank == 0 else 0
    # cov + potrf + (check_limits, k_sov, k_reduce_blocks) + finalize [+ rescale]; int8: + rowscale,
    # lslice, k_sov_oz (memset of the flag is a copy-engine op)
    launches = (1 if (mode in ("dist", "dstore") or rank == 0) else 0) + n_potrf + 3 + 1 + (1 if multi else 0) + \
        (2 if args.sov_method == 1 else 0)
    if mode == "dstore":                       # per phase: one k_sov + one k_rows_copy per rank's piece
        kp = mvn.mvn_potrf_panel_width(n)
        ds = [mvn.dtiles(n, world, r, kp) for r in range(world)]
        for b, e in parallel.sov_phases(-(-n // 128), args.phase_rows):
            launches += 1 + sum(1 for d in ds if mvn.mvn_drows_offset(d, e) > mvn.mvn_drows_offset(d, b))
        launches -= 1                          # the k_sov of the one-shot sweep counted above
    potrf_ms = stage_mean["potrf"]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        # the job (n, N*R of the config) is fixed and split over the GPUs (config D at 8 GPUs: one
        # lattice shift per rank, BASELINE.json): per-GPU work shrinks with N -> strong scaling
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64" if (args.sov_method, args.potrf_method) == (0, 0) else
                 f"f64 (Cholesky as the TLR factorisation at eps = {args.tlr_eps:g}, NEXT-3 R26)" if args.potrf_method == 2 else
                 "f64 (" + " and ".join(x for x, on in [("SOV GEMM (R24)", args.sov_method), ("Cholesky updates (R25)",
                                                        args.potrf_method)] if on) + " as exact int8 tensor-core products)",
        "data": "synthetic",
        "config": config_dict(cfg, world, mode),
        "potrf_mode": mode,
        "cholesky_tflops": (n ** 3 / 3) / (potrf_ms / 1e3) / 1e12,
        "sov_sample_dims_per_s": n * my_samples / (sov_ms / 1e3),
        "region_time_ms": ms_per_step,
        "stage_ms": stage_mean,
        "stage_ms_per_rank": stage_per_rank,
        "sov_method": "int8 tensor cores (NEXT-4, R24)" if args.sov_method == 1 else "fp64 DMMA",
        "potrf_method": {0: "fp64 DMMA", 1: "int8 tensor cores (NEXT-4, R25)",
                         2: f"TLR Cholesky at eps = {args.tlr_eps:g} (NEXT-3, R26)"}[args.potrf_method],
        "roofline": sov_roof,
        "potrf_roofline": {"achieved": (n ** 3 / 3) / (potrf_ms / 1e3) / 1e12, "peak": PEAK_FP64_TFLOPS,
                           "frac": (n ** 3 / 3) / (potrf_ms / 1e3) / 1e12 / PEAK_FP64_TFLOPS,
                           "unit": "TFLOP/s" if args.potrf_method == 0 else
                           "fp64-equivalent TFLOP/s (trailing updates on the int8 tensor cores, R25) over the fp64 peak"
                           if args.potrf_method == 1 else "dense-equivalent TFLOP/s (n^3/3 over the TLR Cholesky time)"},
        "clocks": clk,
        "gpu_launches": launches * args.steps,
        "e2e": e2e,
        "k_star": [int(x) for x in k],
        "qmc_error": qmc_err,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        thr = cpu_threads()
        n_sub, J = oracle_plan(cfg)
        t, t_full, det = oracle_sample(cfg, n_sub, J, thr)
        line["cpu_baseline"] = {"value": n * NR / t_full, "unit": UNIT, "cores": thr, "kind": "oracle",
                                "sample": f"leading {n_sub} of {n} sorted locations x {J} samples of shift 0 "
                                          f"(cov+Cholesky+SOV, {t:.1f} s measured); full-workload time "
                                          f"{t_full:.0f} s extrapolated by op count",
                                "measured": det}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if multi:
        dist.destroy_process_group()
    return 0


def _stdout_json_only():
    """Keep the process's stdout for the one JSON line: native libraries (NCCL's version banner and
    debug lines, CUDA) write to file descriptor 1 directly, so fd 1 is pointed at stderr and Python's
    sys.stdout (where the JSON line is printed) keeps the original stdout."""
    try:
        keep = os.dup(1)
        os.dup2(2, 1)
        sys.stdout = os.fdopen(keep, "w", buffering=1)
    except OSError:
        pass


if __name__ == "__main__":
    _stdout_json_only()
    sys.exit(main())
