"""K1 with a general nu (Temme / CF2 path) at config D's geometry: python tools/k1_nu_time.py [nu] [cfg]."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_14892_b200 as mvn  # noqa: E402
import workloads as W  # noqa: E402

nu = float(sys.argv[1]) if len(sys.argv) > 1 else 1.43391
cfg = W.CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "D"]
inp = W.make_inputs(cfg)
n = cfg.n
d_xy = torch.from_numpy(np.ascontiguousarray(inp.xy)).cuda()
L = mvn.alloc_tiles(n)
ts = []
for it in range(8):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    mvn.mvn_cov_matern(d_xy, cfg.sigma2, cfg.beta, nu, cfg.nugget, out=L)
    e1.record()
    torch.cuda.synchronize()
    if it >= 3:
        ts.append(e0.elapsed_time(e1))
gb = 8.0 * mvn.mvn_tiles_bytes(n) / 8 / 1e9
print(f"cfg={cfg.name} n={n} nu={nu} k1_ms={np.mean(ts):.2f} store_GBps={gb / (np.mean(ts) / 1e3):.0f}", flush=True)
