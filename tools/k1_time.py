"""K1 (k_cov_matern) alone at a BASELINE config: mean of 20 launches with CUDA events, as GB/s of
algorithmic stores (8 n(n+1)/2 bytes... the full lower tiles, padding included) against the HBM peak.
python tools/k1_time.py D   (MVN_K1_VARIANT = 0..4 selects the (rows per thread, CTAs per SM) variant)"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_14892_b200 as mvn  # noqa: E402
import workloads as W  # noqa: E402

cfg = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "D"]
inp = W.make_inputs(cfg)
n = cfg.n
order, a, _ = mvn.mvn_marginal_order(inp.mu, np.full(n, cfg.sigma2 + cfg.nugget), cfg.u)
d_xy = torch.from_numpy(np.ascontiguousarray(inp.xy[order])).cuda()
L = mvn.alloc_tiles(n)
for _ in range(3):
    mvn.mvn_cov_matern(d_xy, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget, out=L)
torch.cuda.synchronize()
ts = []
for _ in range(20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    mvn.mvn_cov_matern(d_xy, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget, out=L)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = float(np.median(ts))
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists("MEASURED_PEAKS.json") else 6442.9
gbs = mvn.mvn_tiles_bytes(n) / (ms / 1e3) / 1e9
print(f"cfg={cfg.name} n={n} variant={os.environ.get("MVN_K1_VARIANT", "0")} k1_ms={ms:.3f} store_GBps={gbs:.0f} "
      f"frac_hbm={gbs / peak:.3f}", flush=True)
