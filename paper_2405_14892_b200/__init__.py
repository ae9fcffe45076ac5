"""paper_2405_14892_b200 — B200-native (sm_100a) confidence-region detection from high-dimensional
MVN probabilities (arXiv 2405.14892), as a thin ctypes binding over libmvn.so (include/mvn.h).

The binding only marshals arguments: every step of the hot path runs in the CUDA library. There
is no CPU fallback — if libmvn.so or an sm_100a device is missing, the calls raise.
PyTorch provides device memory, streams and (in bench.py / parallel.py) torch.distributed.

Function names follow the C ABI (mvn_cov_matern, mvn_potrf, mvn_sov_prefix, ...). Device
arguments are CUDA torch tensors (float64 / int64 / uint64 as documented in include/mvn.h);
host arguments are numpy arrays.
"""
from __future__ import annotations

import atexit
import ctypes
import threading
import math
import os
from dataclasses import dataclass

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libmvn.so")
TILE = 128

MVN_OK, MVN_E_USAGE, MVN_E_NUMERIC, MVN_E_IO, MVN_E_CUDA, MVN_E_NCCL, MVN_E_NOMEM = range(7)
_STATUS = {0: "OK", 1: "USAGE", 2: "NUMERIC", 3: "IO", 4: "CUDA", 5: "NCCL", 6: "NOMEM"}

# every symbol declared in include/mvn.h (tests/test_abi.py checks the header against this list)
ABI_SYMBOLS = [
    "mvn_create", "mvn_destroy", "mvn_set_stream", "mvn_last_error", "mvn_version", "mvn_trim",
    "mvn_tiles_count", "mvn_tiles_bytes", "mvn_pack_lower", "mvn_unpack_lower",
    "mvn_marginal_order", "mvn_cov_matern", "mvn_potrf", "mvn_lattice_generators",
    "mvn_lattice_shifts", "mvn_sov_prefix", "mvn_prefix_rescale", "mvn_prefix_finalize",
    "mvn_confidence_region", "mvn_crd", "mvn_potrf_panel", "mvn_potrf_update", "mvn_panel_pack",
    "mvn_panel_unpack", "mvn_potrf_info", "mvn_mc_validate", "mvn_mc_levels", "mvn_potrf_panel_width",
    "mvn_posterior", "mvn_posterior_tiles", "mvn_tlr_compress",
    "mvn_dtiles_bytes", "mvn_dpanel_numel", "mvn_dcov_matern", "mvn_dpotrf_panel", "mvn_dpanel_pack",
    "mvn_dpotrf_update", "mvn_dgather", "mvn_sov_prefix_ex", "mvn_potrf_ex", "mvn_dpanel_trsm",
    "mvn_sov_prefix_units", "mvn_prefix_reduce", "mvn_sweep_begin", "mvn_sweep_rows", "mvn_sweep_end",
    "mvn_sweep_free", "mvn_drows_offset", "mvn_drows_unpack", "mvn_tlr_slots_bytes", "mvn_tlr_potrf",
    "mvn_sov_prefix_tlr", "mvn_sov_prefix_shifts", "mvn_prefix_shift_stats",
]


class MvnError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"libmvn {_STATUS.get(status, status)}: {msg}")
        self.status = status


class mvn_tiles(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("nb", ctypes.c_int64)]


class mvn_dtiles(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("nb", ctypes.c_int64), ("world", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("kp", ctypes.c_int32), ("prows", ctypes.c_int32)]


class mvn_qmc(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int64), ("R", ctypes.c_int32), ("seed", ctypes.c_uint64),
                ("sample_begin", ctypes.c_int64), ("sample_end", ctypes.c_int64), ("d_gen", ctypes.c_void_p)]


class mvn_mc(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("sample_begin", ctypes.c_int64), ("sample_end", ctypes.c_int64),
                ("method", ctypes.c_int32)]


class mvn_posterior_problem(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("xy", ctypes.c_void_p), ("mu", ctypes.c_void_p), ("m", ctypes.c_int64),
                ("obs", ctypes.c_void_p), ("y", ctypes.c_void_p), ("sigma2", ctypes.c_double),
                ("beta", ctypes.c_double), ("nu", ctypes.c_double), ("nugget", ctypes.c_double),
                ("tau", ctypes.c_double)]


class mvn_crd_problem(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("xy", ctypes.c_void_p), ("mu", ctypes.c_void_p),
                ("sigma2", ctypes.c_double), ("beta", ctypes.c_double), ("nu", ctypes.c_double),
                ("nugget", ctypes.c_double), ("u", ctypes.c_double), ("N", ctypes.c_int64),
                ("R", ctypes.c_int32), ("seed", ctypes.c_uint64), ("conf", ctypes.c_void_p),
                ("nconf", ctypes.c_int64), ("method", ctypes.c_int32), ("tlr_eps", ctypes.c_double)]


class mvn_crd_result(ctypes.Structure):
    _fields_ = [("order", ctypes.c_void_p), ("logP", ctypes.c_void_p), ("k_star", ctypes.c_void_p),
                ("near_tie", ctypes.c_void_p), ("info", ctypes.c_int64), ("ms_stage", ctypes.c_double * 6)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libmvn.so (built by __graft_entry__.build() / _build.py). Raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libmvn.so not built at {LIB_PATH}: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    P, I64, I32, U64, D, S = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64,
                              ctypes.c_double, ctypes.c_int)
    T = mvn_tiles
    sig = {
        "mvn_create": (S, [ctypes.c_int, P, ctypes.POINTER(P)]),
        "mvn_destroy": (None, [P]),
        "mvn_set_stream": (S, [P, P]),
        "mvn_last_error": (ctypes.c_char_p, [P]),
        "mvn_version": (ctypes.c_char_p, []),
        "mvn_trim": (S, [P]),
        "mvn_tiles_count": (I64, [T]),
        "mvn_tiles_bytes": (ctypes.c_size_t, [T]),
        "mvn_pack_lower": (S, [P, T, P, I64, P]),
        "mvn_unpack_lower": (S, [P, T, P, P, I64]),
        "mvn_marginal_order": (S, [I64, P, P, D, P, P, P]),
        "mvn_cov_matern": (S, [P, T, P, D, D, D, D, P]),
        "mvn_potrf": (S, [P, T, P, ctypes.POINTER(I64)]),
        "mvn_lattice_generators": (S, [I64, P]),
        "mvn_lattice_shifts": (S, [U64, I32, I64, P]),
        "mvn_sov_prefix": (S, [P, T, P, P, P, ctypes.POINTER(mvn_qmc), P, P]),
        "mvn_prefix_rescale": (S, [P, I64, P, P, P]),
        "mvn_prefix_finalize": (S, [P, I64, I64, P, P, P]),
        "mvn_confidence_region": (S, [I64, P, P, I64, P, P]),
        "mvn_crd": (S, [P, ctypes.POINTER(mvn_crd_problem), ctypes.POINTER(mvn_crd_result)]),
        "mvn_potrf_panel": (S, [P, T, P, I64, I64]),
        "mvn_potrf_update": (S, [P, T, P, I64, I64, I64, I64, I64, I32]),
        "mvn_potrf_panel_width": (I64, [I64]),
        "mvn_panel_pack": (S, [P, T, P, I64, I64, P]),
        "mvn_panel_unpack": (S, [P, T, P, I64, I64, P]),
        "mvn_potrf_info": (S, [P, ctypes.POINTER(I64), I32]),
        "mvn_mc_validate": (S, [P, T, P, P, ctypes.POINTER(mvn_mc), P, P]),
        "mvn_mc_levels": (S, [I64, P, I64, P, I64, P]),
        "mvn_posterior": (S, [P, ctypes.POINTER(mvn_posterior_problem), P, P, ctypes.POINTER(I64)]),
        "mvn_posterior_tiles": (S, [P, T, P, P]),
        "mvn_tlr_compress": (S, [P, T, P, D, I32, P]),
        "mvn_tlr_slots_bytes": (ctypes.c_size_t, [T, I32]),
        "mvn_tlr_potrf": (S, [P, T, P, D, I32, I32, P, P, P, P, ctypes.POINTER(I64)]),
        "mvn_sov_prefix_tlr": (S, [P, T, P, P, P, P, I32, P, P, ctypes.POINTER(mvn_qmc), P, P]),
        "mvn_sov_prefix_shifts": (S, [P, T, P, P, P, ctypes.POINTER(mvn_qmc), P]),
        "mvn_prefix_shift_stats": (S, [I64, I32, P, P, P]),
        "mvn_dtiles_bytes": (ctypes.c_size_t, [mvn_dtiles]),
        "mvn_dpanel_numel": (I64, [mvn_dtiles, I64]),
        "mvn_dcov_matern": (S, [P, mvn_dtiles, P, D, D, D, D, P]),
        "mvn_dpotrf_panel": (S, [P, mvn_dtiles, P, I64]),
        "mvn_dpanel_pack": (S, [P, mvn_dtiles, P, I64, P]),
        "mvn_dpotrf_update": (S, [P, mvn_dtiles, P, I64, P, I64, I32, I32]),
        "mvn_dgather": (S, [P, mvn_dtiles, P, P]),
        "mvn_dpanel_trsm": (S, [P, mvn_dtiles, P, I64, P]),
        "mvn_sov_prefix_ex": (S, [P, T, P, P, P, ctypes.POINTER(mvn_qmc), I32, P, P]),
        "mvn_potrf_ex": (S, [P, T, P, ctypes.POINTER(I64), I32]),
        "mvn_sov_prefix_units": (S, [P, T, P, P, P, ctypes.POINTER(mvn_qmc), I64, I64, P]),
        "mvn_prefix_reduce": (S, [P, I64, I64, P, P, P]),
        "mvn_sweep_begin": (S, [P, I64, P, P, ctypes.POINTER(mvn_qmc), ctypes.POINTER(P)]),
        "mvn_sweep_rows": (S, [P, P, I64, I64]),
        "mvn_sweep_end": (S, [P, P, P]),
        "mvn_sweep_free": (None, [P]),
        "mvn_drows_offset": (I64, [mvn_dtiles, I64]),
        "mvn_drows_unpack": (S, [P, mvn_dtiles, P, I64, I64, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _np_ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def _dev_ptr(t, dtype=None) -> int:
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda):
        raise TypeError("expected a CUDA torch tensor")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"expected {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return t.data_ptr()


_exiting = False


def _at_exit():
    global _exiting
    _exiting = True                  # process teardown: leave the contexts to the driver


atexit.register(_at_exit)


class Context:
    """An mvn_ctx bound to one CUDA device; follows torch's current stream on every call. One
    context per (thread, device): the stream is context state (mvn_set_stream), so threads must
    not share a context."""

    _tls = threading.local()

    def __init__(self, device: int = 0):
        import torch
        self.device = device
        h = ctypes.c_void_p()
        with torch.cuda.device(device):
            st = lib().mvn_create(device, ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream), ctypes.byref(h))
        if st != MVN_OK:
            raise MvnError(st, f"mvn_create(device={device}) failed (needs a B200 / sm_100 device)")
        self.h = h

    @classmethod
    def get(cls, device: int | None = None, stream=None) -> "Context":
        """The device's context, bound to `stream` (a torch.cuda.Stream) or torch's current stream."""
        import torch
        if device is None:
            device = torch.cuda.current_device()
        by_device = getattr(cls._tls, "by_device", None)
        if by_device is None:
            by_device = cls._tls.by_device = {}
        if device not in by_device:
            by_device[device] = Context(device)
        c = by_device[device]
        st = stream if stream is not None else torch.cuda.current_stream(device)
        lib().mvn_set_stream(c.h, ctypes.c_void_p(st.cuda_stream))
        return c

    def __del__(self):
        # a thread's contexts are collected with its thread-local dict; free their workspace
        h = getattr(self, "h", None)
        if h is not None and _lib is not None and not _exiting:
            try:
                _lib.mvn_destroy(h)
            except Exception:
                pass
            self.h = None

    def check(self, st: int, what: str):
        if st != MVN_OK:
            raise MvnError(st, f"{what}: {lib().mvn_last_error(self.h).decode()}")

    def trim(self):
        self.check(lib().mvn_trim(self.h), "mvn_trim")


def tiles(n: int) -> mvn_tiles:
    return mvn_tiles(n, TILE)


def mvn_tiles_count(n: int) -> int:
    return int(lib().mvn_tiles_count(tiles(n)))


def mvn_tiles_bytes(n: int) -> int:
    return int(lib().mvn_tiles_bytes(tiles(n)))


def alloc_tiles(n: int, device=None):
    import torch
    return torch.empty(mvn_tiles_bytes(n) // 8, dtype=torch.float64, device=device or "cuda")


def mvn_pack_lower(dense, n: int, out=None):
    """dense: (n, n) CUDA float64, read as column-major with ld = n (a C-order tensor's transpose is
    the same memory, and only the lower triangle of a symmetric matrix matters)."""
    c = Context.get(dense.device.index)
    out = alloc_tiles(n, dense.device) if out is None else out
    c.check(lib().mvn_pack_lower(c.h, tiles(n), _dev_ptr(dense), n, _dev_ptr(out)), "mvn_pack_lower")
    return out


def mvn_unpack_lower(t, n: int, out=None):
    """Returns an (n, n) CUDA float64 tensor M whose memory is column-major L, i.e. M.T == L."""
    import torch
    c = Context.get(t.device.index)
    out = torch.zeros((n, n), dtype=torch.float64, device=t.device) if out is None else out
    c.check(lib().mvn_unpack_lower(c.h, tiles(n), _dev_ptr(t), _dev_ptr(out), n), "mvn_unpack_lower")
    return out


def mvn_marginal_order(mu: np.ndarray, var_diag: np.ndarray, u: float):
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    var = np.ascontiguousarray(var_diag, dtype=np.float64)
    n = mu.shape[0]
    order = np.empty(n, dtype=np.int64)
    a = np.empty(n)
    pM = np.empty(n)
    st = lib().mvn_marginal_order(n, _np_ptr(mu), _np_ptr(var), float(u), _np_ptr(order), _np_ptr(a), _np_ptr(pM))
    if st != MVN_OK:
        raise MvnError(st, "mvn_marginal_order")
    return order, a, pM


def mvn_cov_matern(xy_sorted, sigma2: float, beta: float, nu: float, nugget: float, out=None):
    """xy_sorted: (n, 2) CUDA float64 in sorted order. Returns the tile-packed Sigma."""
    import torch
    n = xy_sorted.shape[0]
    c = Context.get(xy_sorted.device.index)
    out = alloc_tiles(n, xy_sorted.device) if out is None else out
    c.check(lib().mvn_cov_matern(c.h, tiles(n), _dev_ptr(xy_sorted, torch.float64), float(sigma2), float(beta),
                                 float(nu), float(nugget), _dev_ptr(out, torch.float64)), "mvn_cov_matern")
    return out


def mvn_potrf(t, n: int, raise_on_numeric: bool = True) -> int:
    """In-place tiled Cholesky. Returns info (-1 ok, else first failing 0-based row)."""
    c = Context.get(t.device.index)
    info = ctypes.c_int64(-1)
    st = lib().mvn_potrf(c.h, tiles(n), _dev_ptr(t), ctypes.byref(info))
    if st == MVN_E_NUMERIC and not raise_on_numeric:
        return int(info.value)
    c.check(st, "mvn_potrf")
    return int(info.value)


POTRF_FP64, POTRF_INT8 = 0, 1


def mvn_potrf_ex(t, n: int, method: int = POTRF_FP64, raise_on_numeric: bool = True) -> int:
    """mvn_potrf with a selectable arithmetic for the trailing updates: POTRF_FP64 (DMMA, default) or
    POTRF_INT8 (the int8 tensor cores, reading R25). Returns info (-1 ok, else the failing row)."""
    c = Context.get(t.device.index)
    info = ctypes.c_int64(-1)
    st = lib().mvn_potrf_ex(c.h, tiles(n), _dev_ptr(t), ctypes.byref(info), int(method))
    if st == MVN_E_NUMERIC and not raise_on_numeric:
        return int(info.value)
    c.check(st, "mvn_potrf_ex")
    return int(info.value)


# ---- NEXT-1: building blocks of the distributed factorisation (driven by parallel.potrf_distributed)
def mvn_potrf_panel_width(n: int) -> int:
    """kp: tile columns per super-panel of mvn_potrf at order n (the distributed schedule uses the same)."""
    return int(lib().mvn_potrf_panel_width(int(n)))


def mvn_potrf_panel(t, n: int, k: int, kp: int = 1, stream=None):
    """Factor tile columns k .. k+kp-1 in place (asynchronous)."""
    c = Context.get(t.device.index, stream)
    c.check(lib().mvn_potrf_panel(c.h, tiles(n), _dev_ptr(t), int(k), int(kp)), "mvn_potrf_panel")


def mvn_potrf_update(t, n: int, k: int, kp: int, col_first: int, col_stride: int = 1, col_block: int = 1,
                     sm_reserve: int = 0, stream=None):
    """A_ij -= sum_{c<kp} L_i,k+c L_j,k+c^T for tile columns j = col_first + m col_stride + b, b < col_block."""
    c = Context.get(t.device.index, stream)
    c.check(lib().mvn_potrf_update(c.h, tiles(n), _dev_ptr(t), int(k), int(kp), int(col_first), int(col_stride),
                                   int(col_block), int(sm_reserve)), "mvn_potrf_update")


def panel_numel(n: int, k: int, kp: int = 1) -> int:
    nt = -(-n // TILE)
    kp = min(kp, nt - k)
    return sum(nt - k - j for j in range(kp)) * TILE * TILE


def mvn_panel_pack(t, n: int, k: int, kp: int, panel, stream=None):
    c = Context.get(t.device.index, stream)
    c.check(lib().mvn_panel_pack(c.h, tiles(n), _dev_ptr(t), int(k), int(kp), _dev_ptr(panel)), "mvn_panel_pack")


def mvn_panel_unpack(panel, n: int, k: int, kp: int, t, stream=None):
    c = Context.get(t.device.index, stream)
    c.check(lib().mvn_panel_unpack(c.h, tiles(n), _dev_ptr(panel), int(k), int(kp), _dev_ptr(t)), "mvn_panel_unpack")


# ---- NEXT-1 distributed storage: a rank's owned tile columns only (include/mvn.h, mvn_dtiles)
def dtiles(n: int, world: int, rank: int, kp: int, prows: int = 1) -> mvn_dtiles:
    """prows = 1: 1-D (column blocks over the ranks); prows = P > 1: 2-D over a P x (world / P) grid."""
    return mvn_dtiles(int(n), TILE, int(world), int(rank), int(kp), int(prows))


def mvn_dtiles_bytes(n: int, world: int, rank: int, kp: int, prows: int = 1) -> int:
    return int(lib().mvn_dtiles_bytes(dtiles(n, world, rank, kp, prows)))


def mvn_dpanel_numel(n: int, world: int, rank: int, kp: int, s: int) -> int:
    return int(lib().mvn_dpanel_numel(dtiles(n, world, rank, kp), int(s)))


def alloc_dtiles(n: int, world: int, rank: int, kp: int, device=None, prows: int = 1):
    import torch
    return torch.empty(max(mvn_dtiles_bytes(n, world, rank, kp, prows) // 8, 1), dtype=torch.float64,
                       device=device or "cuda")


def mvn_dcov_matern(xy_sorted, d: mvn_dtiles, sigma2, beta, nu, nugget, local, stream=None):
    import torch
    c = Context.get(local.device.index, stream)
    c.check(lib().mvn_dcov_matern(c.h, d, _dev_ptr(xy_sorted, torch.float64), float(sigma2), float(beta), float(nu),
                                  float(nugget), _dev_ptr(local, torch.float64)), "mvn_dcov_matern")


def mvn_dpotrf_panel(local, d: mvn_dtiles, s: int, stream=None):
    c = Context.get(local.device.index, stream)
    c.check(lib().mvn_dpotrf_panel(c.h, d, _dev_ptr(local), int(s)), "mvn_dpotrf_panel")


def mvn_dpanel_trsm(local, d: mvn_dtiles, s: int, panel, stream=None):
    c = Context.get(local.device.index, stream)
    c.check(lib().mvn_dpanel_trsm(c.h, d, _dev_ptr(local), int(s), _dev_ptr(panel)), "mvn_dpanel_trsm")


def mvn_dpanel_pack(local, d: mvn_dtiles, s: int, panel, stream=None):
    c = Context.get(local.device.index, stream)
    c.check(lib().mvn_dpanel_pack(c.h, d, _dev_ptr(local), int(s), _dev_ptr(panel)), "mvn_dpanel_pack")


def mvn_dpotrf_update(local, d: mvn_dtiles, s: int, panel, sp_first: int, just_one: bool = False, sm_reserve: int = 0,
                      stream=None):
    c = Context.get(local.device.index, stream)
    c.check(lib().mvn_dpotrf_update(c.h, d, _dev_ptr(local), int(s), _dev_ptr(panel), int(sp_first),
                                    1 if just_one else 0, int(sm_reserve)), "mvn_dpotrf_update")


def mvn_dgather(local, d: mvn_dtiles, full, stream=None):
    c = Context.get(local.device.index, stream)
    c.check(lib().mvn_dgather(c.h, d, _dev_ptr(local), _dev_ptr(full)), "mvn_dgather")


def mvn_potrf_info(device: int = 0, reset: bool = True, stream=None) -> int:
    c = Context.get(device, stream)
    info = ctypes.c_int64(-1)
    c.check(lib().mvn_potrf_info(c.h, ctypes.byref(info), 1 if reset else 0), "mvn_potrf_info")
    return int(info.value)


def mvn_lattice_generators(n: int) -> np.ndarray:
    g = np.empty(n, dtype=np.uint64)
    st = lib().mvn_lattice_generators(n, _np_ptr(g))
    if st != MVN_OK:
        raise MvnError(st, "mvn_lattice_generators")
    return g


def mvn_lattice_shifts(seed: int, R: int, n: int) -> np.ndarray:
    D = np.empty((R, n), dtype=np.uint64)
    st = lib().mvn_lattice_shifts(int(seed), int(R), n, _np_ptr(D))
    if st != MVN_OK:
        raise MvnError(st, "mvn_lattice_shifts")
    return D


def mvn_sov_prefix(L, n: int, a, N: int, R: int, seed: int, begin: int = 0, end: int | None = None,
                   b=None, M=None, S=None, gen=None):
    """One SOV/QMC sweep over global samples [begin, end). Returns CUDA (M, S), n each. gen: optional
    CUDA uint64 (as int64) tensor of n lattice generators replacing R8's table (mvn_qmc.d_gen)."""
    import torch
    c = Context.get(L.device.index)
    end = N * R if end is None else end
    M = torch.empty(n, dtype=torch.float64, device=L.device) if M is None else M
    S = torch.empty(n, dtype=torch.float64, device=L.device) if S is None else S
    q = mvn_qmc(int(N), int(R), int(seed), int(begin), int(end), None if gen is None else _dev_ptr(gen))
    c.check(lib().mvn_sov_prefix(c.h, tiles(n), _dev_ptr(L, torch.float64), _dev_ptr(a, torch.float64),
                                 None if b is None else _dev_ptr(b, torch.float64), ctypes.byref(q),
                                 _dev_ptr(M), _dev_ptr(S)), "mvn_sov_prefix")
    return M, S


def mvn_sov_prefix_shifts(L, n: int, a, N: int, R: int, seed: int, b=None, out=None):
    """log P^(r)_k of every shift r (one sweep per shift): CUDA float64 [R][n]."""
    import torch
    c = Context.get(L.device.index)
    out = torch.empty((R, n), dtype=torch.float64, device=L.device) if out is None else out
    q = mvn_qmc(int(N), int(R), int(seed), 0, int(N) * int(R))
    c.check(lib().mvn_sov_prefix_shifts(c.h, tiles(n), _dev_ptr(L, torch.float64), _dev_ptr(a, torch.float64),
                                        None if b is None else _dev_ptr(b, torch.float64), ctypes.byref(q),
                                        _dev_ptr(out, torch.float64)), "mvn_sov_prefix_shifts")
    return out


def mvn_prefix_shift_stats(logp_shift: np.ndarray):
    """(log P, rel_se) from the per-shift estimates (host, R x n): the combined estimate and the
    relative standard error across the shifts (mvn_prefix_shift_stats)."""
    Ls = np.ascontiguousarray(logp_shift, dtype=np.float64)
    R, n = Ls.shape
    lp, se = np.empty(n), np.empty(n)
    st = lib().mvn_prefix_shift_stats(n, R, _np_ptr(Ls), _np_ptr(lp), _np_ptr(se))
    if st != MVN_OK:
        raise MvnError(st, "mvn_prefix_shift_stats: bad arguments")
    return lp, se


class mvn_sweep:
    """Handle of mvn_sweep_begin (the SOV sweep over row phases, NEXT-1): the samples' log weights and
    Y histories between mvn_sweep_rows calls. Freed by mvn_sweep_end / mvn_sweep_free (or on garbage
    collection)."""

    def __init__(self, h, n: int, device):
        self.h, self.n, self.device = h, n, device
        self.nt = -(-n // TILE)
        self.next = 0

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.mvn_sweep_free(self.h)
            self.h = None


def mvn_sweep_begin(n: int, a, N: int, R: int, seed: int, begin: int = 0, end: int | None = None, b=None,
                    stream=None) -> mvn_sweep:
    import torch
    c = Context.get(a.device.index, stream)
    end = N * R if end is None else end
    q = mvn_qmc(int(N), int(R), int(seed), int(begin), int(end))
    h = ctypes.c_void_p()
    c.check(lib().mvn_sweep_begin(c.h, int(n), _dev_ptr(a, torch.float64),
                                  None if b is None else _dev_ptr(b, torch.float64), ctypes.byref(q),
                                  ctypes.byref(h)), "mvn_sweep_begin")
    return mvn_sweep(h, int(n), a.device)


def mvn_sweep_rows(sw: mvn_sweep, rows, tile_row_begin: int, tile_row_end: int, stream=None):
    """rows: the tiles of tile rows [begin, end) in packed order (tile_rows_slice of a full buffer, or
    a slice assembled from the ranks' storage with mvn_drows_unpack)."""
    import torch
    c = Context.get(sw.device.index, stream)
    if not sw.h:
        raise MvnError(-1, "mvn_sweep_rows: sweep already ended")
    c.check(lib().mvn_sweep_rows(sw.h, _dev_ptr(rows, torch.float64), int(tile_row_begin), int(tile_row_end)),
            "mvn_sweep_rows")
    sw.next = int(tile_row_end)


def mvn_sweep_end(sw: mvn_sweep, M=None, S=None, stream=None):
    """(M, S) of the sweep (as mvn_sov_prefix); frees the handle."""
    import torch
    c = Context.get(sw.device.index, stream)
    M = torch.empty(sw.n, dtype=torch.float64, device=sw.device) if M is None else M
    S = torch.empty(sw.n, dtype=torch.float64, device=sw.device) if S is None else S
    c.check(lib().mvn_sweep_end(sw.h, _dev_ptr(M), _dev_ptr(S)), "mvn_sweep_end")
    sw.h = None
    return M, S


def mvn_sweep_free(sw: mvn_sweep):
    if sw.h:
        Context.get(sw.device.index)
        lib().mvn_sweep_free(sw.h)
        sw.h = None


def tile_rows_range(tile_row_begin: int, tile_row_end: int) -> tuple[int, int]:
    """Element range of tile rows [begin, end) in the full tile-packed buffer."""
    b, e = int(tile_row_begin), int(tile_row_end)
    return b * (b + 1) // 2 * TILE * TILE, e * (e + 1) // 2 * TILE * TILE


def tile_rows_slice(L, tile_row_begin: int, tile_row_end: int):
    lo, hi = tile_rows_range(tile_row_begin, tile_row_end)
    return L[lo:hi]


def mvn_drows_offset(d: mvn_dtiles, tile_row: int) -> int:
    return int(lib().mvn_drows_offset(d, int(tile_row)))


def mvn_drows_unpack(d: mvn_dtiles, piece, tile_row_begin: int, tile_row_end: int, rows, stream=None):
    c = Context.get(rows.device.index, stream)
    c.check(lib().mvn_drows_unpack(c.h, d, _dev_ptr(piece), int(tile_row_begin), int(tile_row_end), _dev_ptr(rows)),
            "mvn_drows_unpack")


SOV_FP64, SOV_INT8 = 0, 1


def mvn_sov_prefix_ex(L, n: int, a, N: int, R: int, seed: int, begin: int = 0, end: int | None = None,
                      b=None, M=None, S=None, method: int = SOV_FP64):
    """mvn_sov_prefix with a selectable GEMM arithmetic: SOV_FP64 (DMMA, default) or SOV_INT8 (the
    update on the int8 tensor cores, reading R24; b must be None)."""
    import torch
    c = Context.get(L.device.index)
    end = N * R if end is None else end
    M = torch.empty(n, dtype=torch.float64, device=L.device) if M is None else M
    S = torch.empty(n, dtype=torch.float64, device=L.device) if S is None else S
    q = mvn_qmc(int(N), int(R), int(seed), int(begin), int(end))
    c.check(lib().mvn_sov_prefix_ex(c.h, tiles(n), _dev_ptr(L, torch.float64), _dev_ptr(a, torch.float64),
                                    None if b is None else _dev_ptr(b, torch.float64), ctypes.byref(q), int(method),
                                    _dev_ptr(M), _dev_ptr(S)), "mvn_sov_prefix_ex")
    return M, S


def sov_units(N: int, R: int) -> int:
    """Number of 128-sample units of N*R samples (mvn_sov_prefix_units)."""
    return -(-int(N) * int(R) // 128)


def mvn_sov_prefix_units(L, n: int, a, N: int, R: int, seed: int, unit_begin: int, unit_end: int, b=None,
                         partial=None):
    """Per-unit partials [unit_end - unit_begin][n][2] (CUDA float64) of the fp64 sweep."""
    import torch
    c = Context.get(L.device.index)
    partial = torch.empty((unit_end - unit_begin, n, 2), dtype=torch.float64, device=L.device) if partial is None else partial
    q = mvn_qmc(int(N), int(R), int(seed), 0, int(N) * int(R))
    c.check(lib().mvn_sov_prefix_units(c.h, tiles(n), _dev_ptr(L, torch.float64), _dev_ptr(a, torch.float64),
                                       None if b is None else _dev_ptr(b, torch.float64), ctypes.byref(q),
                                       int(unit_begin), int(unit_end), _dev_ptr(partial)), "mvn_sov_prefix_units")
    return partial


def mvn_prefix_reduce(partial, M=None, S=None):
    """(M, S) of the unit partials [units][n][2], combined in unit order."""
    import torch
    units, n = partial.shape[0], partial.shape[1]
    c = Context.get(partial.device.index)
    M = torch.empty(n, dtype=torch.float64, device=partial.device) if M is None else M
    S = torch.empty(n, dtype=torch.float64, device=partial.device) if S is None else S
    c.check(lib().mvn_prefix_reduce(c.h, n, units, _dev_ptr(partial), _dev_ptr(M), _dev_ptr(S)), "mvn_prefix_reduce")
    return M, S


def mvn_prefix_rescale(Mglob, M, S):
    c = Context.get(M.device.index)
    c.check(lib().mvn_prefix_rescale(c.h, M.numel(), _dev_ptr(Mglob), _dev_ptr(M), _dev_ptr(S)), "mvn_prefix_rescale")


def mvn_prefix_finalize(M, S, NR: int, out=None):
    import torch
    c = Context.get(M.device.index)
    out = torch.empty_like(M) if out is None else out
    c.check(lib().mvn_prefix_finalize(c.h, M.numel(), int(NR), _dev_ptr(M), _dev_ptr(S), _dev_ptr(out)),
            "mvn_prefix_finalize")
    return out


def mvn_confidence_region(logP: np.ndarray, conf):
    lp = np.ascontiguousarray(logP, dtype=np.float64)
    cf = np.ascontiguousarray(conf, dtype=np.float64)
    k = np.empty(len(cf), dtype=np.int64)
    tie = np.empty(len(cf), dtype=np.int32)
    st = lib().mvn_confidence_region(lp.shape[0], _np_ptr(lp) if lp.size else None, _np_ptr(cf) if cf.size else None,
                                     len(cf), _np_ptr(k) if cf.size else None, _np_ptr(tie) if cf.size else None)
    if st != MVN_OK:
        raise MvnError(st, "mvn_confidence_region")
    return k, tie.astype(bool)


# ---- NEXT-2: Monte-Carlo validation of the regions
def mvn_mc_validate(L, n: int, a, seed: int, begin: int, end: int, count=None, first=None, method: int = 0):
    """Draws samples [begin, end) of mu + L z (reading R20) and accumulates the histogram of their
    first failing rows into `count` (CUDA uint64, n+1; created zeroed if None). `first`: optional
    CUDA int32 of end-begin, receives f_s. method 0: X = L Z on fp64 DMMA; 1: on the int8 tensor
    cores (tcgen05, Ozaki split, R22). Returns count."""
    import torch
    c = Context.get(L.device.index)
    if count is None:
        count = torch.zeros(n + 1, dtype=torch.uint64, device=L.device)
    m = mvn_mc(int(seed), int(begin), int(end), int(method))
    c.check(lib().mvn_mc_validate(c.h, tiles(n), _dev_ptr(L, torch.float64), _dev_ptr(a, torch.float64), ctypes.byref(m),
                                  _dev_ptr(count, torch.uint64), None if first is None else _dev_ptr(first, torch.int32)),
            "mvn_mc_validate")
    return count


def mvn_mc_levels(count: np.ndarray, N_total: int, k_star) -> np.ndarray:
    """p_hat(k*) = #{f >= k*} / N_total (host)."""
    cnt = np.ascontiguousarray(count, dtype=np.uint64)
    ks = np.ascontiguousarray(k_star, dtype=np.int64)
    out = np.empty(len(ks))
    st = lib().mvn_mc_levels(cnt.shape[0] - 1, _np_ptr(cnt), int(N_total), _np_ptr(ks) if ks.size else None, len(ks),
                             _np_ptr(out) if ks.size else None)
    if st != MVN_OK:
        raise MvnError(st, "mvn_mc_levels")
    return out


# ---- NEXT-4: posterior conditioning (Eq. 7-8)
def mvn_posterior(xy, mu, obs, y, sigma2, beta, nu, nugget, tau, device: int = 0):
    """Returns host (mu_post, var_post); Sigma_post stays in the context for mvn_posterior_tiles."""
    xy = np.ascontiguousarray(xy, dtype=np.float64)
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    obs = np.ascontiguousarray(obs, dtype=np.int64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    n, m = mu.shape[0], obs.shape[0]
    c = Context.get(device)
    mp, vp = np.empty(n), np.empty(n)
    info = ctypes.c_int64(-1)
    prob = mvn_posterior_problem(n, _np_ptr(xy), _np_ptr(mu), m, _np_ptr(obs), _np_ptr(y), float(sigma2), float(beta),
                                 float(nu), float(nugget), float(tau))
    c.check(lib().mvn_posterior(c.h, ctypes.byref(prob), _np_ptr(mp), _np_ptr(vp), ctypes.byref(info)), "mvn_posterior")
    return mp, vp


def mvn_posterior_tiles(order: np.ndarray, out=None, device: int = 0):
    """Sigma_post of the last mvn_posterior, permuted to `order`, as a tile-packed CUDA tensor."""
    order = np.ascontiguousarray(order, dtype=np.int64)
    n = order.shape[0]
    c = Context.get(device)
    out = alloc_tiles(n, f"cuda:{device}") if out is None else out
    c.check(lib().mvn_posterior_tiles(c.h, tiles(n), _np_ptr(order), _dev_ptr(out)), "mvn_posterior_tiles")
    return out


def crd_posterior(xy, mu, obs, y, sigma2, beta, nu, nugget, tau, u, N, R, seed, conf, device: int = 0):
    """Alg. 1 on the posterior field: condition (Eq. 7-8), order by the posterior marginals,
    factor Sigma_post in sorted order, one SOV sweep, regions. Every step runs in libmvn."""
    import torch
    mp, vp = mvn_posterior(xy, mu, obs, y, sigma2, beta, nu, nugget, tau, device)
    order, a, _ = mvn_marginal_order(mp, vp, u)
    T = mvn_posterior_tiles(order, device=device)
    n = mp.shape[0]
    info = mvn_potrf(T, n)
    d_a = torch.from_numpy(a).to(f"cuda:{device}")
    M, S = mvn_sov_prefix(T, n, d_a, N, R, seed)
    logp = mvn_prefix_finalize(M, S, N * R).cpu().numpy()
    k, tie = mvn_confidence_region(logp, conf)
    return CrdOutput(order, logp, k, tie, info, ()), mp, vp, T


# ---- NEXT-3 (part): fixed-accuracy TLR compression
TLR_ABS, TLR_REL_FRO = 0, 1


def mvn_tlr_compress(t, n: int, eps: float, ranks=None, mode: int = TLR_ABS):
    """Replaces every off-diagonal tile of the tile-packed `t` by its truncated SVD, in place: mode
    TLR_ABS keeps sigma_i >= eps, TLR_REL_FRO the smallest rank with ||A - A_k||_F <= eps ||A||_F.
    Returns the CUDA int32 ranks, tile (I, J) at I(I-1)/2 + J."""
    import torch
    c = Context.get(t.device.index)
    nt = -(-n // TILE)
    ranks = torch.empty(max(nt * (nt - 1) // 2, 1), dtype=torch.int32, device=t.device) if ranks is None else ranks
    c.check(lib().mvn_tlr_compress(c.h, tiles(n), _dev_ptr(t, torch.float64), float(eps), int(mode),
                                   _dev_ptr(ranks, torch.int32)),
            "mvn_tlr_compress")
    return ranks


@dataclass
class TlrFactor:
    """mvn_tlr_potrf's outputs besides the factor itself (in the tile buffer): the factor slots of
    the off-diagonal tiles (U_t, V_t: [tiles][kmax columns][128] views of 128 x kmax column-major
    blocks), the ranks of L~ and of Sigma~, and info."""
    U: object
    V: object
    ranks: object
    ranks_sigma: object
    kmax: int
    info: int


def mvn_sov_prefix_tlr(L, f: "TlrFactor", n: int, a, N: int, R: int, seed: int, begin: int = 0,
                       end: int | None = None, b=None, M=None, S=None):
    """mvn_sov_prefix with the factored update s = sum_J U_TJ (V_TJ^T Y_J) from mvn_tlr_potrf's factor
    slots (f); L supplies the dense diagonal tiles. Returns CUDA (M, S)."""
    import torch
    c = Context.get(L.device.index)
    end = N * R if end is None else end
    M = torch.empty(n, dtype=torch.float64, device=L.device) if M is None else M
    S = torch.empty(n, dtype=torch.float64, device=L.device) if S is None else S
    q = mvn_qmc(int(N), int(R), int(seed), int(begin), int(end))
    c.check(lib().mvn_sov_prefix_tlr(c.h, tiles(n), _dev_ptr(L, torch.float64), _dev_ptr(f.U, torch.float64),
                                     _dev_ptr(f.V, torch.float64), _dev_ptr(f.ranks, torch.int32), int(f.kmax),
                                     _dev_ptr(a, torch.float64), None if b is None else _dev_ptr(b, torch.float64),
                                     ctypes.byref(q), _dev_ptr(M), _dev_ptr(S)), "mvn_sov_prefix_tlr")
    return M, S


def mvn_tlr_potrf(t, n: int, eps: float, mode: int = TLR_ABS, kmax: int = TILE, raise_on_numeric: bool = True,
                  U=None, V=None) -> TlrFactor:
    """TLR Cholesky in place (reading R26): Sigma's off-diagonal tiles compressed at eps, the tile
    columns factored with the updates in factored form, every L tile truncated at eps once; on
    return `t` holds L~ (dense diagonal tiles, off-diagonal tiles U V^T reconstructed for the dense
    SOV)."""
    import torch
    c = Context.get(t.device.index)
    nt = -(-n // TILE)
    noff = nt * (nt - 1) // 2
    if U is None:
        U = torch.empty((max(noff, 1), kmax, TILE), dtype=torch.float64, device=t.device)
    if V is None:
        V = torch.empty((max(noff, 1), kmax, TILE), dtype=torch.float64, device=t.device)
    ranks = torch.zeros(max(noff, 1), dtype=torch.int32, device=t.device)
    ranks_s = torch.zeros(max(noff, 1), dtype=torch.int32, device=t.device)
    info = ctypes.c_int64(-1)
    st = lib().mvn_tlr_potrf(c.h, tiles(n), _dev_ptr(t, torch.float64), float(eps), int(mode), int(kmax),
                             _dev_ptr(U, torch.float64), _dev_ptr(V, torch.float64), _dev_ptr(ranks, torch.int32),
                             _dev_ptr(ranks_s, torch.int32), ctypes.byref(info))
    if not (st == MVN_E_NUMERIC and not raise_on_numeric):
        c.check(st, "mvn_tlr_potrf")
    return TlrFactor(U, V, ranks, ranks_s, kmax, int(info.value))


@dataclass
class CrdOutput:
    order: np.ndarray
    logP: np.ndarray
    k_star: np.ndarray
    near_tie: np.ndarray
    info: int
    ms_stage: tuple


CRD_SOV_INT8, CRD_POTRF_INT8, CRD_TLR = 1, 2, 4


def mvn_crd(xy: np.ndarray, mu: np.ndarray, sigma2, beta, nu, nugget, u, N, R, seed, conf, device: int = 0,
            pinned_out=None, method: int = 0, tlr_eps: float = 0.0) -> CrdOutput:
    """End-to-end Alg. 1 through the C ABI with HOST buffers (upload, a1..a10, download).
    method: 0 fp64; bit 0 the SOV GEMM on the int8 tensor cores, bit 1 the Cholesky updates too;
    bit 2 (CRD_TLR) the TLR Cholesky at accuracy tlr_eps (NEXT-3)."""
    xy = np.ascontiguousarray(xy, dtype=np.float64)
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    cf = np.ascontiguousarray(conf, dtype=np.float64)
    n = mu.shape[0]
    c = Context.get(device)
    order = np.empty(n, dtype=np.int64)
    logP = np.empty(n)
    k = np.empty(max(len(cf), 1), dtype=np.int64)
    tie = np.empty(max(len(cf), 1), dtype=np.int32)
    prob = mvn_crd_problem(n, _np_ptr(xy), _np_ptr(mu), sigma2, beta, nu, nugget, u, int(N), int(R), int(seed),
                           _np_ptr(cf) if cf.size else None, len(cf), int(method), float(tlr_eps))
    res = mvn_crd_result(_np_ptr(order), _np_ptr(logP), _np_ptr(k), _np_ptr(tie), -1)
    c.check(lib().mvn_crd(c.h, ctypes.byref(prob), ctypes.byref(res)), "mvn_crd")
    return CrdOutput(order, logP, k[:len(cf)], tie[:len(cf)].astype(bool), int(res.info), tuple(res.ms_stage))


__all__ = [n for n in dir() if n.startswith("mvn_")] + ["Context", "MvnError", "lib", "TILE", "alloc_tiles", "dtiles",
                                                      "alloc_dtiles"]
