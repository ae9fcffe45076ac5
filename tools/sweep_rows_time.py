"""Time the SOV sweep over row phases (mvn_sweep_*, NEXT-1) against the one-shot mvn_sov_prefix on a
BASELINE config: python tools/sweep_rows_time.py D [samples] [phase_rows ...].
samples: the sweep's sample range [0, samples) (default: all N*R; a rank's shard at W GPUs is
N*R/W). Each phase is run two ways: on a view of the full factor (no copy: the cost of cutting the
sweep), and on a staging buffer the phase's rows are first copied into (the arrival of the rows:
what sov_distributed's assembly adds on the compute stream). Checks bitwise equality of (M, S).
Every variant: one warm-up run, then the best of 2."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_14892_b200 as mvn  # noqa: E402
import workloads as W  # noqa: E402

cfg = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "D"]
ns = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "-" else cfg.NR
prs = [int(x) for x in sys.argv[3:]] or [8, 32]
inp = W.make_inputs(cfg)
n, nt = cfg.n, -(-cfg.n // 128)
order, a, _ = mvn.mvn_marginal_order(inp.mu, np.full(n, cfg.sigma2 + cfg.nugget), cfg.u)
L = mvn.mvn_cov_matern(torch.from_numpy(np.ascontiguousarray(inp.xy[order])).cuda(), cfg.sigma2, cfg.beta, cfg.nu,
                       cfg.nugget)
assert mvn.mvn_potrf(L, n) == -1
d_a = torch.from_numpy(a).cuda()


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), out


REPS = 2


def best(fn):
    fn()                                         # warm-up (first-use allocations)
    ts, out = [], None
    for _ in range(REPS):
        t, out = timed(fn)
        ts.append(t)
    return min(ts), out


t0, (M0, S0) = best(lambda: mvn.mvn_sov_prefix(L, n, d_a, cfg.N, cfg.R, cfg.seed_lattice, 0, ns))
flop = n * (n - 1) * ns
print(f"cfg={cfg.name} samples={ns} one-shot sov_ms={t0:.1f} frac={flop / (t0 / 1e3) / 1e12 / 37.07:.3f}", flush=True)
for pr in prs:
    phases = [(b, min(b + pr, nt)) for b in range(0, nt, pr)]
    stage = None
    for mode in ("view", "staged"):
        if mode == "staged":
            mx = max(mvn.tile_rows_range(b, e)[1] - mvn.tile_rows_range(b, e)[0] for b, e in phases)
            stage = torch.empty(mx, dtype=torch.float64, device="cuda")

        def run():
            sw = mvn.mvn_sweep_begin(n, d_a, cfg.N, cfg.R, cfg.seed_lattice, 0, ns)
            for b, e in phases:
                rows = mvn.tile_rows_slice(L, b, e)
                if stage is not None:
                    s = stage[:rows.numel()]
                    s.copy_(rows)
                    rows = s
                mvn.mvn_sweep_rows(sw, rows, b, e)
            return mvn.mvn_sweep_end(sw)
        t, (M, S) = best(run)
        same = bool(torch.equal(M, M0) and torch.equal(S, S0))
        print(f"  phase_rows={pr} phases={len(phases)} {mode}: sov_ms={t:.1f} ({t / t0:.3f}x) "
              f"frac={flop / (t / 1e3) / 1e12 / 37.07:.3f} bitwise={same}", flush=True)
