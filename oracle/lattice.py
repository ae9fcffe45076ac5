"""ORACLE (test infrastructure only) — the QMC point set, reading R8 of DESIGN.md.

The paper calls its sampler QMC while Alg. 2 line 4 draws
R(i,j) ~ U(0,1); BASELINE.json fixes "Richtmyer-lattice QMC points (sqrt-prime generators) with
seeded random shifts". Defined exactly in integers so both sides can produce identical bits:

    p_k   = the k-th prime (p_1 = 2), assigned to sorted position k = 1..n
    G_k   = floor(frac(sqrt(p_k)) * 2^64) = isqrt(p_k << 128) mod 2^64
    D_k^r = SplitMix64 output function applied to seed + GAMMA * (r * 2^32 + k + 1)   (mod 2^64)
    X     = (j * G_k + D_k^r) mod 2^64,  j = 1..N
    w     = (floor(X / 2^12) + 1/2) * 2^-52

Everything here is exact Python integer arithmetic (obviously correct, independent of the CUDA
library's own implementation, which tests compare bit for bit).
"""
from __future__ import annotations

import math

import numpy as np

MASK64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15  # SplitMix64 increment (golden ratio * 2^64, odd)


def primes(n: int) -> list[int]:
    """First n primes: sieve of Eratosthenes up to the Rosser bound p_n < n (ln n + ln ln n) (n >= 6)."""
    if n <= 0:
        return []
    bound = 15 if n < 6 else int(n * (math.log(n) + math.log(math.log(n)))) + 1
    is_p = np.ones(bound + 1, dtype=bool)
    is_p[:2] = False
    for c in range(2, math.isqrt(bound) + 1):
        if is_p[c]:
            is_p[c * c:: c] = False
    out = [int(p) for p in np.flatnonzero(is_p)[:n]]
    assert len(out) == n
    return out


def generators(n: int) -> np.ndarray:
    """G_k = floor(frac(sqrt(p_k)) 2^64) for k = 1..n, as uint64 (reading R8)."""
    return np.array([math.isqrt(p << 128) & MASK64 for p in primes(n)], dtype=np.uint64)


def splitmix64_mix(z: int) -> int:
    """SplitMix64 output function (Steele, Lea, Flood 2014; the finaliser of java.util.SplittableRandom)."""
    z &= MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def shifts(seed: int, R: int, n: int) -> np.ndarray:
    """D[r][k] = mix(seed + GAMMA*(r*2^32 + k + 1)) for r < R, k < n, as uint64 (reading R8)."""
    D = np.empty((R, n), dtype=np.uint64)
    for r in range(R):
        D[r] = [splitmix64_mix(seed + GAMMA * ((r << 32) + k + 1)) for k in range(n)]
    return D


def lattice_w(j: int, G: int, D: int) -> float:
    """w for lattice index j (1-based) of a row with generator G and shift D."""
    X = (j * int(G) + int(D)) & MASK64
    return ((X >> 12) + 0.5) * 2.0 ** -52
