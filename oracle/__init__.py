"""oracle -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct CPU reference for arXiv:1903.06681's hot path
(spatially / hybrid sample-spatial partitioned 2D convolution). Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this package; the product package paper_1903_06681_b200 never
does, and this package never imports it.

  * oracle.c      : Eqs. 1-3 and BN statistics, fp64 NCHW
  * partition.py  : blocked distributions, brute-force halo dependence sets,
                    explicit halo slicing
  * perfmodel.py  : the paper's cost formulas

Every function cites the passage it follows. fp64 unless stated.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (-O2, OpenMP, no fast-math: IEEE fp64)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fno-fast-math", "-fPIC", "-shared",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        i64, dp = ctypes.c_int64, ctypes.POINTER(ctypes.c_double)
        L.oracle_conv_fwd.argtypes = [i64] * 8 + [dp, dp, dp, i64, i64]
        L.oracle_conv_bwd_data.argtypes = [i64] * 8 + [dp, dp, dp, i64, i64]
        L.oracle_conv_bwd_filter.argtypes = [i64] * 8 + [dp, dp, dp]
        L.oracle_conv_bwd_filter_entry.argtypes = [i64] * 8 + [dp, dp] + [i64] * 4
        L.oracle_conv_bwd_filter_entry.restype = ctypes.c_double
        L.oracle_bn_stats.argtypes = [i64] * 4 + [dp, dp, dp]
        L.oracle_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def out_extent(H: int, K: int, S: int, P: int) -> int:
    """H~ = floor((H + 2P - K)/S) + 1 (reading R2; equals SPEC.md:45's ceil form)."""
    return (H + 2 * P - K) // S + 1


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def conv_fwd(x, w, S: int = 1, P: int | None = None, rows=None) -> np.ndarray:
    """Eq. 1, stride/pad generalised (R2). x: N,C,H,W; w: F,C,K,K.
    rows=(i0,i1) restricts the computed output rows (others left zero)."""
    x, w = _f64(x), _f64(w)
    N, C, H, W = x.shape
    F, C2, K, K2 = w.shape
    assert C2 == C and K2 == K
    P = K // 2 if P is None else P
    Ho, Wo = out_extent(H, K, S, P), out_extent(W, K, S, P)
    y = np.zeros((N, F, Ho, Wo))
    i0, i1 = rows or (0, Ho)
    lib().oracle_conv_fwd(N, C, H, W, F, K, S, P, _p(x), _p(w), _p(y), i0, i1)
    return y


def conv_bwd_data(dy, w, H: int, W: int, S: int = 1, P: int | None = None, rows=None) -> np.ndarray:
    """Eq. 3, strided adjoint form (R4). Returns dx: N,C,H,W."""
    dy, w = _f64(dy), _f64(w)
    N, F, Ho, Wo = dy.shape
    F2, C, K, _ = w.shape
    assert F2 == F
    P = K // 2 if P is None else P
    assert (Ho, Wo) == (out_extent(H, K, S, P), out_extent(W, K, S, P))
    dx = np.zeros((N, C, H, W))
    u0, u1 = rows or (0, H)
    lib().oracle_conv_bwd_data(N, C, H, W, F, K, S, P, _p(dy), _p(w), _p(dx), u0, u1)
    return dx


def conv_bwd_filter(x, dy, K: int, S: int = 1, P: int | None = None) -> np.ndarray:
    """Eq. 2, i,j over the output extent (R3). Returns dw: F,C,K,K."""
    x, dy = _f64(x), _f64(dy)
    N, C, H, W = x.shape
    F = dy.shape[1]
    P = K // 2 if P is None else P
    assert dy.shape == (N, F, out_extent(H, K, S, P), out_extent(W, K, S, P))
    dw = np.zeros((F, C, K, K))
    lib().oracle_conv_bwd_filter(N, C, H, W, F, K, S, P, _p(x), _p(dy), _p(dw))
    return dw


def conv_bwd_filter_entry(x, dy, K: int, S: int, P: int, f: int, c: int, a: int, b: int) -> float:
    """One entry of Eq. 2 (for sampled parity at full size)."""
    x, dy = _f64(x), _f64(dy)
    N, C, H, W = x.shape
    F = dy.shape[1]
    return float(lib().oracle_conv_bwd_filter_entry(N, C, H, W, F, K, S, P, _p(x), _p(dy), f, c, a, b))


def bn_stats(t) -> tuple[np.ndarray, np.ndarray]:
    """Per-channel mean and biased variance over (n,h,w), two-pass
    (reading R11)."""
    t = _f64(t)
    N, C, H, W = t.shape
    mean, var = np.zeros(C), np.zeros(C)
    lib().oracle_bn_stats(N, C, H, W, _p(t), _p(mean), _p(var))
    return mean, var
