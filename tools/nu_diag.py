import sys, numpy as np, torch, mpmath as mp
sys.path.insert(0, '.')
import paper_2405_14892_b200 as mvn, oracle
sys.path.insert(0, 'tests')
from test_gpu_parity import to_dense_lower
mp.mp.dps = 30
for nu, beta, n in [(0.3, 0.05, 300), (1.00003, 0.1, 300), (1.43391, 0.1, 400)]:
    xy = np.random.default_rng(int(nu * 1000) + n).uniform(size=(n, 2))
    T = mvn.mvn_cov_matern(torch.from_numpy(xy).cuda(), 1.3, beta, nu, 1e-8)
    G = to_dense_lower(T, n)
    S = oracle.covariance(xy, 1.3, beta, nu, 1e-8)
    low = np.tril(S, -1)
    rel = np.where(low > 1e-280, np.abs(G - low) / np.maximum(np.abs(low), 1e-300), 0)
    idx = np.argsort(rel.ravel())[::-1][:4]
    for t in idx:
        i, j = divmod(t, n)
        h = mp.sqrt(mp.mpf(xy[i,0]-xy[j,0])**2 + mp.mpf(xy[i,1]-xy[j,1])**2)
        x = h / beta
        ref = 1.3 / (2**(mp.mpf(nu)-1) * mp.gamma(nu)) * x**nu * mp.besselk(nu, x)
        print(f"nu={nu} x={float(x):.4g} gpu_rel={float(abs(G[i,j]-ref)/ref):.2e} oracle_rel={float(abs(S[i,j]-ref)/ref):.2e}")
