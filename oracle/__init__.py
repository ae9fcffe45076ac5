"""ORACLE — test infrastructure only.

A plain, slow, obviously-correct CPU implementation of the hot path of arXiv 2405.14892
(dense confidence-region detection: Matérn covariance -> Cholesky -> one SOV/QMC sweep giving
every prefix probability P_k -> regions). It exists to prove the CUDA path right.

Rules:
  * Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
    ``--impl reference`` legs may import, call, link or execute anything under ``oracle/``.
  * It shares no code with ``paper_2405_14892_b200/`` (no kernels, headers, helpers, tables or
    constant generators) and neither imports the other. Only ``workloads/`` (seeded input
    synthesis, none of the method's arithmetic) serves both.
  * fp64 throughout; every function cites the PAPER.md passage (``P:n`` = line n of
    /root/reference/PAPER.md) or the DESIGN.md reading (R1..R18) it follows.

Parity pins: every function here is pinned by ``tests/test_oracle_*.py`` (``-m "not gpu"``)
against closed forms, library special functions, brute force or paper values. None is
"parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "csrc", "oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the C oracle (plain -O2, no fast-math, no FMA contraction, OpenMP for independent work)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-shared", "-fPIC",
               "-std=c11", "-o", _LIB_PATH + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB_PATH + ".tmp", _LIB_PATH)
    return _LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        d, i64, u64p, dp, i = ctypes.c_double, ctypes.c_longlong, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int
        for name, res, args in [
            ("orc_Phi", d, [d]), ("orc_Phibar", d, [d]), ("orc_erfcx_far", d, [d]),
            ("orc_log_Phibar_far", d, [d]), ("orc_Phiinv_lower", d, [d]),
            ("orc_Phibar_inv_far", d, [d, d]), ("orc_lattice_w", d, [ctypes.c_uint64] * 3),
            ("orc_sov_step", None, [d, d, d, dp, dp]),
            ("orc_cholesky", i64, [i64, dp, i]),
            ("orc_sov_unit", i, [i64, dp, i64, dp, dp, u64p, u64p, i64, i64, dp, dp, dp]),
            ("orc_sov_units", i, [i64, dp, i64, dp, dp, u64p, u64p, i64, i64, i64, i64, i64, dp, i]),
            ("orc_mc_mix", ctypes.c_uint64, [ctypes.c_uint64] * 3),
            ("orc_mc_z", d, [ctypes.c_uint64] * 3),
            ("orc_mc_first", i, [i64, dp, i64, dp, ctypes.c_uint64, i64, i64, dp, dp, dp, i]),
        ]:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def ptr(a: np.ndarray) -> int:
    return a.ctypes.data


from .lattice import primes, generators, shifts, splitmix64_mix, lattice_w  # noqa: E402
from .matern import matern, covariance  # noqa: E402
from .pipeline import (  # noqa: E402
    Phi, Phibar, Phiinv, sov_step, cholesky, marginal_order, sov_units, sov_unit,
    combine_units, prefix_logp, per_shift_logp, shift_stats, region, crd, crd_cov,
)
from .mcval import mc_z, mc_first, mc_counts, mc_levels  # noqa: E402
from .posterior import posterior, posterior_field  # noqa: E402
from .tlr import tlr_compress, compress_tile, tlr_cholesky  # noqa: E402
