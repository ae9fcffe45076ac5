"""Seeded synthetic inputs for the BASELINE.json configurations (shared by oracle and CUDA path).

This module holds NONE of the method's arithmetic: no Matérn evaluation, no Cholesky, no
Phi / Phi^{-1}, no lattice. It only produces the inputs both sides read:

  * geometry: a g x g grid of cell centres ((i+1/2)/g, (j+1/2)/g) on [0,1]^2, original index
    i*g + j, plus independent uniform jitter U(-0.4/g, +0.4/g) per coordinate (BASELINE configs:
    "regular grid on [0,1]^2 with uniform jitter +-0.4/g (seeded)"). Stands in for the paper's
    ExaGeoStat synthetic fields and the wind data, neither of which is in the
    container.
  * mean field mu: "one seeded draw from the same GP" (BASELINE). Synthesised with J random
    Fourier features of the Matérn spectral density (reading R15 in DESIGN.md): for the paper's
    parametrisation C(h) = s2 (h/b)^nu K_nu(h/b) / (2^(nu-1) Gamma(nu)) (Eq. 6, no sqrt(2 nu)), the
    2-D spectral density is proportional to (1 + b^2 |w|^2)^-(nu+1), i.e. w = z / (b sqrt(g)) with
    z ~ N(0, I_2), g ~ chi^2_(2 nu); mu(x) = sqrt(2 s2 / J) sum_j cos(w_j . x + phi_j),
    phi_j ~ U(0, 2 pi). Marginally ~N(0, s2), spatially smooth at range b; it costs O(n J) and
    needs no factorisation, so it scales to n = 102,400.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    g: int                 # grid side; n = g*g
    sigma2: float
    beta: float
    nu: float
    nugget: float
    u: float
    N: int                 # lattice points per shift
    R: int                 # random shifts
    conf: tuple            # confidence levels 1 - alpha
    seed_geom: int
    seed_mu: int
    seed_lattice: int
    gpus: tuple = (1,)

    @property
    def n(self) -> int:
        return self.g * self.g

    @property
    def NR(self) -> int:
        return self.N * self.R


_LEVELS4 = (0.80, 0.90, 0.95, 0.99)
_LEVELS50 = tuple(t / 100.0 for t in range(50, 100))   # conf_t = t/100 from integers (R16)

CONFIGS = {
    "A": Config("A", 20, 1.0, 0.1, 0.5, 1e-8, 0.0, 10_000, 10, _LEVELS4, 1001, 2001, 3001, (1,)),
    "B": Config("B", 70, 1.0, 0.1, 0.5, 1e-8, 0.0, 10_000, 10, _LEVELS4, 1002, 2002, 3002, (1, 2)),
    "C": Config("C", 128, 1.0, 0.05, 1.5, 1e-8, 0.5, 20_000, 10, _LEVELS4, 1003, 2003, 3003, (1, 2, 4, 8)),
    "D": Config("D", 256, 1.0, 0.03, 0.5, 1e-8, 0.0, 10_000, 8, _LEVELS4, 1004, 2004, 3004, (1, 2, 4, 8)),
    "E": Config("E", 320, 1.0, 0.02, 1.5, 1e-8, 0.0, 50_000, 8, _LEVELS50, 1005, 2005, 3005, (1, 2, 4, 8)),
}


def jittered_grid(g: int, seed: int) -> np.ndarray:
    """n x 2 float64 locations, original index i*g + j."""
    rng = np.random.default_rng(seed)
    i, j = np.meshgrid(np.arange(g), np.arange(g), indexing="ij")
    xy = np.stack([(i.ravel() + 0.5) / g, (j.ravel() + 0.5) / g], axis=1)
    xy += rng.uniform(-0.4 / g, 0.4 / g, size=xy.shape)
    return xy


def gp_mean_draw(xy: np.ndarray, sigma2: float, beta: float, nu: float, seed: int, J: int = 2048) -> np.ndarray:
    """One seeded random-Fourier-feature draw of a zero-mean Matérn GP at xy (see module doc)."""
    rng = np.random.default_rng(seed)
    z = rng.standard_normal((J, 2))
    gch = rng.chisquare(2.0 * nu, size=J)
    omega = z / (beta * np.sqrt(gch))[:, None]
    phase = rng.uniform(0.0, 2.0 * np.pi, size=J)
    amp = np.sqrt(2.0 * sigma2 / J)
    mu = np.empty(xy.shape[0])
    step = 8192
    for s in range(0, xy.shape[0], step):
        mu[s:s + step] = amp * np.cos(xy[s:s + step] @ omega.T + phase).sum(axis=1)
    return mu


@dataclass
class Inputs:
    cfg: Config
    xy: np.ndarray      # n x 2, original order
    mu: np.ndarray      # n, original order
    extra: dict = field(default_factory=dict)


def make_inputs(cfg: Config | str) -> Inputs:
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    xy = jittered_grid(cfg.g, cfg.seed_geom)
    mu = gp_mean_draw(xy, cfg.sigma2, cfg.beta, cfg.nu, cfg.seed_mu)
    return Inputs(cfg, xy, mu)


def small_config(name: str, g: int, N: int, R: int, base: str = "A", **kw) -> Config:
    """A scaled-down variant of a BASELINE config (same kernel family), for fast parity tests."""
    c = CONFIGS[base]
    d = dict(c.__dict__)
    d.update(name=name, g=g, N=N, R=R, **kw)
    return Config(**d)


@dataclass
class PosteriorInputs:
    cfg: Config
    xy: np.ndarray
    mu: np.ndarray          # prior mean (0, the paper's choice "mu = 0")
    obs: np.ndarray         # m distinct observed site indices (sorted)
    y: np.ndarray           # m noisy observations
    tau: float


def make_posterior_inputs(cfg: Config | str, m: int, tau: float = 0.5, seed: int = 4242) -> PosteriorInputs:
    """NEXT-4 workload (§V-A: "6,250 samples under the additive noise N(0, 0.5^2)
    ... randomly selected"): the config's jittered grid, a zero prior mean, a hidden field drawn
    from the same GP (random Fourier features, as for mu), m sites chosen uniformly without
    replacement, y = field + N(0, tau^2) noise. Seeded; no method arithmetic."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    xy = jittered_grid(cfg.g, cfg.seed_geom)
    field_ = gp_mean_draw(xy, cfg.sigma2, cfg.beta, cfg.nu, seed)
    rng = np.random.default_rng(seed + 1)
    obs = np.sort(rng.choice(xy.shape[0], size=m, replace=False)).astype(np.int64)
    y = field_[obs] + tau * rng.standard_normal(m)
    return PosteriorInputs(cfg, xy, np.zeros(xy.shape[0]), obs, y, tau)
