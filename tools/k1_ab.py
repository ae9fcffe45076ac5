"""K1 A/B: python tools/k1_ab.py <package root> [cfg]: mean of 20 k_cov_matern launches (CUDA events)
with the libmvn of the package under <package root> (e.g. an older build copied aside)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, sys.argv[1])
sys.path.insert(1, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_14892_b200 as mvn  # noqa: E402
import workloads as W  # noqa: E402

cfg = W.CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "D"]
inp = W.make_inputs(cfg)
n = cfg.n
order, a, _ = mvn.mvn_marginal_order(inp.mu, np.full(n, cfg.sigma2 + cfg.nugget), cfg.u)
d_xy = torch.from_numpy(np.ascontiguousarray(inp.xy[order])).cuda()
L = mvn.alloc_tiles(n)
ts = []
for it in range(25):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    mvn.mvn_cov_matern(d_xy, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget, out=L)
    e1.record()
    torch.cuda.synchronize()
    if it >= 5:
        ts.append(e0.elapsed_time(e1))
print(f"{sys.argv[1]} cfg={cfg.name} k1_ms={np.mean(ts):.3f} min={np.min(ts):.3f} {mvn.__file__}", flush=True)
