"""CPU checks of constants compiled into the CUDA kernels (host-side, no GPU):
the AS 241 (PPND16) coefficients of Phi_inv_lower in normal.cuh reproduce Phi^{-1} to <= 1e-15
relative over [1e-300, 0.5] when evaluated exactly as the kernel does (Horner, fp64)."""
import math
import os
import re

import mpmath as mp
import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = open(os.path.join(ROOT, "paper_2405_14892_b200", "csrc", "normal.cuh")).read()


def _blocks():
    body = SRC[SRC.index("double Phi_inv_lower"):SRC.index("// General limits")]
    nums = [float(x) for x in re.findall(r"[0-9]\.[0-9]+e[+-]?[0-9]+", body)]
    # order in the source: region 1 num (8), den (7 + 1.0 literal), region 2 num, den, region 3 num, den
    return nums


def horner_src(coefs_hi_to_lo, r):
    s = coefs_hi_to_lo[0]
    for c in coefs_hi_to_lo[1:]:
        s = s * r + c
    return s


def ppnd16(p, C):
    a1, b1, a2, b2, a3, b3 = C
    q = p - 0.5
    if abs(q) <= 0.425:
        r = 0.180625 - q * q
        return q * horner_src(a1, r) / horner_src(b1 + [1.0], r)
    r = math.sqrt(-math.log(p))
    if r <= 5.0:
        r -= 1.6
        return -horner_src(a2, r) / horner_src(b2 + [1.0], r)
    r -= 5.0
    return -horner_src(a3, r) / horner_src(b3 + [1.0], r)


def test_ppnd16_coefficients_in_kernel():
    nums = _blocks()
    assert len(nums) == 6 * 8 - 3, len(nums)      # each denominator ends in the literal 1.0
    C, i = [], 0
    for blk in range(3):
        C.append(nums[i:i + 8]); i += 8
        C.append(nums[i:i + 7]); i += 7
    mp.mp.dps = 40
    worst = 0.0
    for p in list(np.logspace(-300, -1, 300)) + list(np.linspace(0.1, 0.5, 100)):
        lo, hi = mp.mpf(-40), mp.mpf(0.1)
        for _ in range(200):
            mid = (lo + hi) / 2
            if mp.log(mp.ncdf(mid)) < mp.log(p):
                lo = mid
            else:
                hi = mid
        want = float((lo + hi) / 2)
        got = ppnd16(float(p), C)
        # p = 0.5: the bisection returns ~1e-41 for the exact 0; compare absolutely below 1e-20
        worst = max(worst, abs(got - want) / max(abs(want), 1e-20))
    assert worst <= 1e-15, worst


def test_far_tail_threshold_consistent_with_oracle():
    k = float(re.search(r"kFarTail = ([0-9.]+)", SRC).group(1))
    osrc = open(os.path.join(ROOT, "oracle", "csrc", "oracle.c")).read()
    assert float(re.search(r"#define ORC_FAR_TAIL ([0-9.]+)", osrc).group(1)) == k == 35.0


def test_branch_free_ppnd16_uses_same_coefficients():
    """Phi_inv_lower_nb (the SOV fast path) selects per lane among the same AS 241 coefficient sets
    as Phi_inv_lower (pinned above against mpmath)."""
    ref = _blocks()
    C, i = [], 0
    for blk in range(3):
        C.append(ref[i:i + 8]); i += 8
        C.append(ref[i:i + 7]); i += 7
    body = SRC[SRC.index("double Phi_inv_lower_nb"):SRC.index("// Upper-exceedance fast path")]
    nums = [float(x) for x in re.findall(r"[0-9]\.[0-9]+e[+-]?[0-9]+", body)]
    assert nums[:8] == C[0] and nums[8:15] == C[1]
    sel = nums[15:]
    assert sel[0:16:2] == C[2] and sel[1:16:2] == C[4]          # numerator: (r <= 5, r > 5) pairs
    assert sel[16:30:2] == C[3] and sel[17:30:2] == C[5]        # denominator
