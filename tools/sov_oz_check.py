"""GPU check of the int8 SOV (mvn_sov_prefix_ex, MVN_SOV_INT8) against the fp64 sweep and the
oracle (shared L), small to large n; prints max |dlog P| and timings. Run under `timeout`."""
import math
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2405_14892_b200 as mvn  # noqa: E402
import workloads as W  # noqa: E402


def logp(M, S, NR):
    M, S = M.cpu().numpy(), S.cpu().numpy()
    with np.errstate(divide="ignore"):
        return np.where(S > 0, M + np.log(S) - math.log(NR), -np.inf)


def case(name, g, N, R, base, oracle_check=True, begin=0, end=None):
    cfg = W.small_config(name, g, N, R, base=base) if g else W.CONFIGS[base]
    inp = W.make_inputs(cfg)
    n = cfg.n
    order, a, _ = mvn.mvn_marginal_order(inp.mu, np.full(n, cfg.sigma2 + cfg.nugget), cfg.u)
    d_xy = torch.from_numpy(np.ascontiguousarray(inp.xy[order])).cuda()
    d_a = torch.from_numpy(a).cuda()
    T = mvn.mvn_cov_matern(d_xy, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget)
    assert mvn.mvn_potrf(T, n) == -1
    end = cfg.NR if end is None else end
    out = {}
    for meth in (0, 1):
        ts = []
        for it in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            M, S = mvn.mvn_sov_prefix_ex(T, n, d_a, cfg.N, cfg.R, cfg.seed_lattice, begin, end, method=meth)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        out[meth] = (logp(M, S, end - begin), min(ts))
    d = np.max(np.abs(out[0][0] - out[1][0]))
    flops = float(n) * (n - 1) * (end - begin)
    line = (f"{name}: n={n} samples={end - begin} max|dlogP| int8-fp64 = {d:.3e}; fp64 {out[0][1]*1e3:.1f} ms "
            f"({flops / out[0][1] / 1e12:.1f} TF), int8 {out[1][1]*1e3:.1f} ms ({flops / out[1][1] / 1e12:.1f} fp64-eq TF)")
    if oracle_check:
        import oracle
        from oracle import lattice
        L = mvn.mvn_unpack_lower(T, n).T.contiguous().cpu().numpy()
        G, D = lattice.generators(n), lattice.shifts(cfg.seed_lattice, cfg.R, n)
        parts = oracle.sov_units(L, a, np.full(n, np.inf), G, D, cfg.N, cfg.R, cfg.N, nthreads=0)
        Mo, So = oracle.combine_units(parts)
        lo = oracle.prefix_logp(Mo, So, cfg.NR)
        line += f"; vs oracle: fp64 {np.max(np.abs(out[0][0] - lo)):.3e}, int8 {np.max(np.abs(out[1][0] - lo)):.3e}"
    print(line, flush=True)


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "small"
    torch.cuda.set_device(0)
    if which == "small":
        case("n100", 10, 200, 2, "A")            # one row block: no MMA
        case("n144", 12, 200, 2, "A")            # two row blocks
        case("n400", 20, 1000, 4, "A")
        case("n1024", 32, 1000, 4, "C")
        case("n2500", 50, 1000, 2, "B")
    elif which == "mid":
        case("n4900", 70, 2000, 4, "B")
        case("n10000", 100, 2000, 2, "C", oracle_check=False)
    else:
        for c in which.split(","):
            case(c, None, None, None, c, oracle_check=False)
