"""Time the SOV sweep alone (CUDA events) on a BASELINE config: python tools/sov_time.py C [reps].
Environment knobs of libmvn are read once per process (MVN_SOV_LAG, MVN_SOV_HINTS), so A/B runs
use separate processes."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_14892_b200 as mvn  # noqa: E402
import workloads as W  # noqa: E402

cfg = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
if len(sys.argv) > 4:                                    # reduced variant: grid side g, total samples N*R
    g, NR = int(sys.argv[3]), int(sys.argv[4])
    cfg = W.small_config(f"{cfg.name}-g{g}", g, NR // cfg.R, cfg.R, base=cfg.name)
inp = W.make_inputs(cfg)
n = cfg.n
order, a, _ = mvn.mvn_marginal_order(inp.mu, np.full(n, cfg.sigma2 + cfg.nugget), cfg.u)
L = mvn.mvn_cov_matern(torch.from_numpy(np.ascontiguousarray(inp.xy[order])).cuda(), cfg.sigma2, cfg.beta, cfg.nu,
                       cfg.nugget)
assert mvn.mvn_potrf(L, n) == -1
d_a = torch.from_numpy(a).cuda()
ts = []
for it in range(reps + 1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    M, S = mvn.mvn_sov_prefix(L, n, d_a, cfg.N, cfg.R, cfg.seed_lattice)
    e1.record()
    torch.cuda.synchronize()
    if it:
        ts.append(e0.elapsed_time(e1))
lp = mvn.mvn_prefix_finalize(M, S, cfg.NR).cpu().numpy()
ms = float(np.mean(ts)) if ts else float("nan")
fr = n * (n - 1) * cfg.NR / (ms / 1e3) / 1e12 / 37.07
print(f"cfg={cfg.name} lag={os.environ.get('MVN_SOV_LAG', 'def')} serial={os.environ.get('MVN_SOV_SERIAL', 'def')} "
      f"sov_ms={ms:.1f} frac={fr:.3f} logP[-1]={lp[-1]:.12f} logP[100]={lp[min(100, n - 1)]:.15f}", flush=True)
