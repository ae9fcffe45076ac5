"""TLR rank structure vs tile size and ordering (tooling, CPU, numpy SVD): the paper's rank figure
 uses 980-wide tiles; the path's tiles are 128 wide and Alg. 1 factors Sigma in the
marginal-probability order (R1). For n = g^2 sites (exponential kernel, the three correlation
levels of P:368) this prints the mean / max rank of the off-diagonal tiles at eps = 1e-3 relative
to the tile width, in the sorted order and in the spatial (grid row-major) order.
Run: PYTHONPATH=. python tools/tlr_rank_vs_tile.py [g]
(Study tool: its own few lines of Eq. 6 and the sort key; it does not use oracle/.)"""
import sys

import numpy as np

import workloads as W


def covariance(xy, sigma2, beta, nu, nugget):
    """Eq. 6 for nu = 1/2 (the exponential kernel of these settings), dense fp64 (study tool)."""
    assert nu == 0.5
    h = np.sqrt(((xy[:, None, :] - xy[None, :, :]) ** 2).sum(-1))
    return sigma2 * np.exp(-h / beta) + nugget * np.eye(len(xy))


def marginal_order(mu, var, u):
    """Descending marginal exceedance probability = descending (mu - u) / sqrt(var), stable (R13)."""
    return np.argsort(-(mu - u) / np.sqrt(var), kind="stable"), None, None


def ranks(S, nb, eps):
    n = S.shape[0]
    nt = n // nb
    out = []
    for I in range(1, nt):
        for J in range(I):
            s = np.linalg.svd(S[I * nb:(I + 1) * nb, J * nb:(J + 1) * nb], compute_uv=False)
            out.append(int(np.count_nonzero(s >= eps)))
    return np.array(out)


def main(g=70, eps=1e-3):
    print(f"n = {g * g}, eps = {eps}")
    print("| beta | tile | order | mean rank / tile | max rank / tile |")
    print("|---|---|---|---|---|")
    for beta in (0.033, 0.1, 0.234):
        cfg = W.small_config("rk", g, 10, 1, base="B", beta=beta)
        inp = W.make_inputs(cfg)
        order, _, _ = marginal_order(inp.mu, np.full(cfg.n, cfg.sigma2 + cfg.nugget), cfg.u)
        for nb in (128, 490, 980):
            if cfg.n // nb < 2:
                continue
            for name, idx in (("sorted", order), ("spatial", np.arange(cfg.n))):
                S = covariance(inp.xy[idx], cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget)
                r = ranks(S, nb, eps)
                print(f"| {beta} | {nb} | {name} | {r.mean():.0f} / {nb} ({r.mean() / nb:.0%}) | {r.max()} / {nb} |", flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 70)
