"""Design study for kernels_tlr.cu (tooling, not product): sweeps of the round-robin one-sided Jacobi
iteration (same pairing, same 1e-15 relative test, same floor) on Matérn tiles of a config-C-like
covariance in sorted order, applied to A directly vs to R^T of a column-pivoted QR of A, and the
resulting ||A - A_k||_2 vs sigma_{k+1} (Eckart-Young). numpy emulation, vectorised per step.
Run: PYTHONPATH=. python tools/tlr_jacobi_sweeps.py"""
import numpy as np
import scipy.linalg as sl

import workloads as W


def covariance(xy, sigma2, beta, nu, nugget):
    """Eq. 6 for nu = 3/2 (config C's kernel), dense fp64 (study tool; does not use oracle/)."""
    assert nu == 1.5
    h = np.sqrt(((xy[:, None, :] - xy[None, :, :]) ** 2).sum(-1)) / beta
    return sigma2 * (1.0 + h) * np.exp(-h) + nugget * np.eye(len(xy))

NB = 128


def rr(pos, s):
    return 0 if pos == 0 else 1 + (pos - 1 + s) % (NB - 1)


PAIRS = [(np.array([rr(p, s) for p in range(64)]), np.array([rr(NB - 1 - p, s) for p in range(64)])) for s in range(NB - 1)]


def jacobi(X, eps, max_sweeps):
    """Columns of X orthogonalised in place; returns (sweeps run, X)."""
    C = X.T.copy()
    f2 = 1e-6 * eps * eps
    for sw in range(max_sweeps):
        changed = False
        for ci, cj in PAIRS:
            x, y = C[ci], C[cj]
            al, be, ga = (x * x).sum(1), (y * y).sum(1), (x * y).sum(1)
            m = (np.abs(ga) > 1e-15 * np.sqrt(al * be)) & (ga != 0) & (al + be >= f2)
            if m.any():
                changed = True
                z = (be[m] - al[m]) / (2 * ga[m])
                t = np.where(z >= 0, 1.0, -1.0) / (np.abs(z) + np.sqrt(1 + z * z))
                c = 1 / np.sqrt(1 + t * t)
                sn = c * t
                xm, ym = x[m], y[m]
                C[ci[m]] = c[:, None] * xm - sn[:, None] * ym
                C[cj[m]] = sn[:, None] * xm + c[:, None] * ym
        if not changed:
            return sw + 1, C.T
    return max_sweeps, C.T


def main(eps=1e-6, max_sweeps=60):
    cfg = W.small_config("tlr30", 30, 100, 1, base="C")
    inp = W.make_inputs(cfg)
    order = np.argsort(-(inp.mu - cfg.u), kind="stable")          # R13 sort key (equal variances)
    S = covariance(inp.xy[order], cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget)
    for (I, J) in [(1, 0), (2, 0), (3, 1), (4, 0), (6, 5)]:
        A = S[I * NB:(I + 1) * NB, J * NB:(J + 1) * NB]
        s = np.linalg.svd(A, compute_uv=False)
        sw_a, Xa = jacobi(A, eps, max_sweeps)
        _, R, P = sl.qr(A, pivoting=True)
        sw_r, Xr = jacobi(R.T.copy(), eps, max_sweeps)
        sig = np.sqrt((Xr * Xr).sum(0))
        keep = np.where(sig >= eps)[0]
        V = np.zeros((NB, len(keep)))
        V[P, :] = Xr[:, keep] / sig[keep]
        err = np.linalg.norm(A - A @ V @ V.T, 2)
        print(f"tile ({I},{J}): sweeps on A {sw_a:2d}, on R^T {sw_r:2d}; k {len(keep)}, "
              f"||A - A_k||_2 {err:.4e} vs sigma_k+1 {s[len(keep)]:.4e}")


if __name__ == "__main__":
    main()
