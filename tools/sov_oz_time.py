"""Time the int8 SOV sweep (mvn_sov_prefix_ex, MVN_SOV_INT8) alone at a BASELINE config (CUDA
events, mean of reps after one warm-up); MVN_SOV_OZ_LAG (cluster lockstep) is read once per process.
python tools/sov_oz_time.py D [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_14892_b200 as mvn  # noqa: E402
import workloads as W  # noqa: E402

cfg = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "D"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
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
    M, S = mvn.mvn_sov_prefix_ex(L, n, d_a, cfg.N, cfg.R, cfg.seed_lattice, method=1)
    e1.record()
    torch.cuda.synchronize()
    if it:
        ts.append(e0.elapsed_time(e1))
lp = mvn.mvn_prefix_finalize(M, S, cfg.NR).cpu().numpy()
ms = float(np.mean(ts))
print(f"cfg={cfg.name} lag={os.environ.get('MVN_SOV_OZ_LAG', '0')} int8_sov_ms={ms:.1f} "
      f"fp64eq_tf={n * (n - 1) * cfg.NR / (ms / 1e3) / 1e12:.1f} logP[-1]={lp[-1]:.10f}", flush=True)
