"""Latency of the Cholesky at small n (CUDA events, median of 20): python tools/potrf_small_time.py.
n = 128 is one diagonal tile (k_potrf_diag2 alone); the others add the TRSM / update chain."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_14892_b200 as mvn  # noqa: E402

for n in [128, 256, 400, 1024, 2048, 4900]:
    xy = torch.from_numpy(np.random.default_rng(n).uniform(size=(n, 2))).cuda()
    S = mvn.mvn_cov_matern(xy, 1.0, 0.1, 0.5, 1e-8)
    L = torch.empty_like(S)
    ts = []
    for it in range(23):
        L.copy_(S)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        assert mvn.mvn_potrf(L, n) == -1
        e1.record()
        torch.cuda.synchronize()
        if it >= 3:
            ts.append(e0.elapsed_time(e1))
    nt = -(-n // 128)
    ms = float(np.median(ts))
    print(f"n={n} tiles={nt} potrf_ms={ms:.3f} per_tile_column_us={ms * 1e3 / nt:.1f} kp={mvn.mvn_potrf_panel_width(n)}",
          flush=True)
