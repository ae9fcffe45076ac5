"""NEXT-3 accuracy study (§VI-B, P:434-439 and Fig. 6 ranks): dense vs fixed-accuracy
TLR-compressed covariance through the same CUDA path (POTRF -> SOV -> regions), on the paper's three
synthetic settings: n = 40,000 sites, exponential kernel (nu = 1/2), sigma^2 = 1, range beta = 0.033
(weak), 0.1 (medium), 0.234 (strong) (Fig. 5 captions). Inputs: jittered 200 x 200 grid, GP
mean draw (workloads.gp_mean_draw), u = 0, N*R = 10,000 x 8. Every step runs in libmvn; no oracle.
TLR_CHOL=1 (round 2): the TLR Cholesky itself (mvn_tlr_potrf, R26: Sigma compressed, updates in
factored form, every L tile truncated at eps) instead of the dense POTRF of the compressed Sigma.
Prints one JSON object per (beta, eps) and writes gpurun_out/tlr_study[_chol]_mode<m>.json."""
import json
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_14892_b200 as mvn  # noqa: E402
import workloads as W  # noqa: E402

NB = 128
CONF = (0.80, 0.90, 0.95, 0.99)


def rank_stats(r):
    r = np.asarray(r)
    return {"mean": float(r.mean()), "median": float(np.median(r)), "p90": float(np.percentile(r, 90)),
            "max": int(r.max()), "zero_frac": float(np.mean(r == 0)),
            "hist": np.bincount(np.minimum(r, 128) // 16, minlength=9).tolist()}


def run(T, n, a, N, R, seed):
    info = mvn.mvn_potrf(T, n, raise_on_numeric=False)
    if info != -1:
        return info, None
    d_a = torch.from_numpy(a).cuda()
    M, S = mvn.mvn_sov_prefix(T, n, d_a, N, R, seed)
    logp = mvn.mvn_prefix_finalize(M, S, N * R).cpu().numpy()
    return info, logp


def main():
    g = int(os.environ.get("TLR_G", "200"))
    N, R = int(os.environ.get("TLR_N", "10000")), int(os.environ.get("TLR_R", "8"))
    betas = [float(b) for b in os.environ.get("TLR_BETAS", "0.033,0.1,0.234").split(",")]
    epss = [float(e) for e in os.environ.get("TLR_EPS", "1e-1,1e-2,1e-3,1e-4").split(",")]
    mode = int(os.environ.get("TLR_MODE", "0"))          # 0: sigma_i >= eps, 1: relative Frobenius per tile
    chol = os.environ.get("TLR_CHOL", "0") == "1"
    out = []
    for beta in betas:
        cfg = W.small_config(f"tlr_b{beta}", g, N, R, base="B", beta=beta)
        inp = W.make_inputs(cfg)
        n = cfg.n
        order, a, _ = mvn.mvn_marginal_order(inp.mu, np.full(n, cfg.sigma2 + cfg.nugget), cfg.u)
        d_xs = torch.from_numpy(np.ascontiguousarray(inp.xy[order])).cuda()
        base = mvn.mvn_cov_matern(d_xs, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget)
        T = base.clone()
        t0 = time.time()
        info, lp_d = run(T, n, a, N, R, cfg.seed_lattice)
        torch.cuda.synchronize()
        k_d = mvn.mvn_confidence_region(lp_d, CONF)[0]
        rec = {"beta": beta, "n": n, "eps": 0.0, "info": info, "k_star": [int(x) for x in k_d],
               "s_dense": time.time() - t0}
        print(json.dumps(rec), flush=True)
        out.append(rec)
        # ranks in the spatial (grid row-major) order, for context: Fig. 6 compresses the
        # matrix of the geometry's own ordering
        d_xy = torch.from_numpy(np.ascontiguousarray(inp.xy)).cuda()
        for eps in epss:
            Tg = mvn.mvn_cov_matern(d_xy, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget)
            rg = mvn.mvn_tlr_compress(Tg, n, eps, mode=mode).cpu().numpy()
            del Tg
            T.copy_(base)
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if chol:
                ev0.record()
                f = mvn.mvn_tlr_potrf(T, n, eps, mode=mode, raise_on_numeric=False)
                ev1.record()
                torch.cuda.synchronize()
                ms = ev0.elapsed_time(ev1)
                ranks, info = f.ranks_sigma.cpu().numpy(), f.info
                lp = None
                if info == -1:
                    M, S = mvn.mvn_sov_prefix(T, n, torch.from_numpy(a).cuda(), N, R, cfg.seed_lattice)
                    lp = mvn.mvn_prefix_finalize(M, S, N * R).cpu().numpy()
                rec = {"beta": beta, "n": n, "eps": eps, "mode": mode, "tlr_potrf_ms": ms, "info": info,
                       "ranks_sorted_order": rank_stats(ranks), "ranks_L": rank_stats(f.ranks.cpu().numpy()),
                       "ranks_spatial_order": rank_stats(rg)}
                del f
            else:
                ev0.record()
                ranks = mvn.mvn_tlr_compress(T, n, eps, mode=mode)
                ev1.record()
                torch.cuda.synchronize()
                ms = ev0.elapsed_time(ev1)
                ranks = ranks.cpu().numpy()
                info, lp = run(T, n, a, N, R, cfg.seed_lattice)
                rec = {"beta": beta, "n": n, "eps": eps, "mode": mode, "compress_ms": ms, "info": info,
                       "ranks_sorted_order": rank_stats(ranks), "ranks_spatial_order": rank_stats(rg)}
            if lp is not None:
                k = mvn.mvn_confidence_region(lp, CONF)[0]
                P_d, P_t = np.exp(lp_d), np.exp(lp)
                fin = np.isfinite(lp_d) & np.isfinite(lp) & (lp_d > math.log(0.5))
                rec.update({"k_star": [int(x) for x in k], "dk_star": [int(x - y) for x, y in zip(k, k_d)],
                            "max_abs_dP": float(np.max(np.abs(P_t - P_d))),
                            "max_abs_dlogP_P_gt_half": float(np.max(np.abs(lp[fin] - lp_d[fin]))) if fin.any() else None})
            print(json.dumps(rec), flush=True)
            out.append(rec)
        del T, base
        torch.cuda.empty_cache()
    os.makedirs("gpurun_out", exist_ok=True)
    with open(f"gpurun_out/tlr_study{'_chol' if chol else ''}_mode{mode}.json", "w") as fo:
        json.dump(out, fo, indent=1)


if __name__ == "__main__":
    main()
