"""Time mvn_potrf alone (CUDA events) on a BASELINE config: python tools/potrf_time.py D [reps] [grid] [method].
method 1 = the trailing updates on the int8 tensor cores (mvn_potrf_ex); prints the residual on
sampled entries against the fp64 factor too.
MVN_POTRF_KP (super-panel width) is read once per process, so A/B runs use separate processes."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_14892_b200 as mvn  # noqa: E402
import workloads as W  # noqa: E402

cfg = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "D"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
method = int(sys.argv[4]) if len(sys.argv) > 4 else 0
if len(sys.argv) > 3 and sys.argv[3] != "-":             # grid side override: n = g^2
    cfg = W.small_config(f"{cfg.name}-g{sys.argv[3]}", int(sys.argv[3]), cfg.N, cfg.R, base=cfg.name)
inp = W.make_inputs(cfg)
n = cfg.n
order, a, _ = mvn.mvn_marginal_order(inp.mu, np.full(n, cfg.sigma2 + cfg.nugget), cfg.u)
d_xy = torch.from_numpy(np.ascontiguousarray(inp.xy[order])).cuda()
L = mvn.alloc_tiles(n)
ts = []
for it in range(reps + 1):
    mvn.mvn_cov_matern(d_xy, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget, out=L)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    info = mvn.mvn_potrf_ex(L, n, method)
    e1.record()
    torch.cuda.synchronize()
    assert info == -1
    if it:
        ts.append(e0.elapsed_time(e1))
ms = float(np.mean(ts))
extra = ""
if method:
    R = mvn.alloc_tiles(n)
    mvn.mvn_cov_matern(d_xy, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget, out=R)
    mvn.mvn_potrf(R, n)
    extra = f" max|L_int8 - L_fp64|={float((L - R).abs().max()):.3e}"
print(f"cfg={cfg.name} n={n} method={method} kp={os.environ.get('MVN_POTRF_KP', 'def')} potrf_ms={ms:.1f} "
      f"tflops={n ** 3 / 3 / (ms / 1e3) / 1e12:.2f} frac={n ** 3 / 3 / (ms / 1e3) / 1e12 / 37.07:.3f}{extra}", flush=True)
