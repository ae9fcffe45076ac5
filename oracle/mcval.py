"""ORACLE (test infrastructure only) — NEXT-2, Monte-Carlo validation of the confidence regions.

PAPER.md §V-C1: "This algorithm draws N samples from the fitted distribution, where N_s
represents the number of samples exceeding a given threshold. The MC estimate of the confidence
probability is then expressed as p_hat(alpha) = N_s/N, and it is expected that
p_hat(alpha) ~ 1 - alpha"; supplement P:20-23 ("to verify the estimated confidence region has
correct confidence levels, we draw N samples from the fitted distribution and let N_s denote the
number of samples larger than the threshold").

Reading R20: sample s draws z_k = Phi^{-1}(w_{k,s}) with w from the SplitMix64 output
function of seed + GAMMA (s 2^32 + k + 1) (the counter construction of the lattice shifts, R8);
the field in sorted order is mu + L z, so it exceeds u on the region o(1..k*) iff
(L z)_k > a_k for every k < k*. One pass per sample gives its first failing row f, and
p_hat(k*) = #{s : f_s >= k*} / N for every level at once.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import lib, ptr


def mc_z(seed: int, s: int, k: int) -> float:
    """z_{k,s} (reading R20), computed by the C oracle (its own mix and Halley Phi^{-1})."""
    return lib().orc_mc_z(int(seed), int(s), int(k))


def mc_first(L: np.ndarray, a: np.ndarray, seed: int, s0: int, ns: int, nthreads: int = 0, diagnostics=False):
    """First failing row of samples s0 .. s0+ns-1 (n if none). L: row-major lower (n x n)."""
    L = np.ascontiguousarray(L, dtype=np.float64)
    a = np.ascontiguousarray(a, dtype=np.float64)
    n = L.shape[0]
    first = np.empty(ns, dtype=np.int32)
    margin = np.empty(ns)
    gap = np.empty(ns)
    err = lib().orc_mc_first(n, ptr(L), n, ptr(a), int(seed), int(s0), int(ns), ptr(first), ptr(margin),
                             ptr(gap), int(nthreads))
    assert err == 0
    return (first, margin, gap) if diagnostics else first


def mc_counts(first: np.ndarray, n: int) -> np.ndarray:
    """count[f] = number of samples whose first failing row is f (f = 0..n)."""
    return np.bincount(np.asarray(first, dtype=np.int64), minlength=n + 1).astype(np.int64)


def mc_levels(count: np.ndarray, k_star, N: int) -> np.ndarray:
    """p_hat(k*) = #{f >= k*} / N for each region size k* (P:595)."""
    tail = np.cumsum(np.asarray(count, dtype=np.int64)[::-1])[::-1]     # tail[k] = #{f >= k}
    return np.array([tail[int(k)] / N for k in k_star])
