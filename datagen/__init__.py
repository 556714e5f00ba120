"""Seeded, counter-based synthetic input generator shared by the oracle side and
the CUDA side of the tests and of bench.py.

This module holds NO arithmetic of the method (no convolution, no halo, no
statistics): it only maps (seed, tensor_id, global NCHW linear index) to a
value, so that every rank's shard and the oracle's global tensor see the same
numbers whatever the decomposition (SURVEY.md §8(d) "Concrete synthetic
inputs"; DESIGN.md §3 "Input recipe").

Value grids (chosen so bf16 rounding is exact and both sides consume the same
numbers):
  * "act"   (x, dy): k/128 - 1, k = h & 255          -> {-1, ..., 127/128}
  * "weight" (w)   : the same grid * 2^-ceil(log2(sqrt(C*K*K)))  (power of
                     two, so still bf16-exact; keeps |y| ~ O(1))
  * "act24"        : 24-bit uniform grid in [-1, 1)   (fp32-exact, not bf16)

splitmix64 is the public-domain mixer of Steele/Lea/Flood (2014); the key is
splitmix64(seed ^ (tensor_id << 32)) + index.
"""
from __future__ import annotations

import math

import numpy as np

SEED = 1903
TID_X, TID_W, TID_DY = 0, 1, 2

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _key(seed: int, tensor_id: int) -> np.uint64:
    k = np.array([(seed ^ (tensor_id << 32)) & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64)
    return _splitmix64(k)[0]


def hash_index(seed: int, tensor_id: int, index: np.ndarray) -> np.ndarray:
    """64-bit hash of global linear indices (uint64 array)."""
    with np.errstate(over="ignore"):
        return _splitmix64(index.astype(np.uint64) + _key(seed, tensor_id))


def weight_scale(C: int, K: int) -> float:
    """2^-ceil(log2(sqrt(C*K*K))): a power of two, so scaled values stay bf16-exact."""
    return 2.0 ** (-math.ceil(math.log2(math.sqrt(C * K * K))))


def _values(h: np.ndarray, kind: str) -> np.ndarray:
    if kind in ("act", "weight"):
        return (h & np.uint64(255)).astype(np.float64) / 128.0 - 1.0
    if kind == "act24":
        return (h >> np.uint64(40)).astype(np.float64) / float(1 << 23) - 1.0
    raise ValueError(f"unknown kind {kind!r}")


def gen_block(shape, seed: int, tensor_id: int, kind: str = "act",
              n=None, c=None, h=None, w=None, scale: float = 1.0) -> np.ndarray:
    """Values of the global NCHW tensor of `shape` restricted to the index
    ranges n, c, h, w (each a (lo, hi) half-open pair or None for all).
    Returned as float64 NCHW of the block's extents."""
    N, C, H, W = shape
    rn = np.arange(*(n or (0, N)), dtype=np.uint64)
    rc = np.arange(*(c or (0, C)), dtype=np.uint64)
    rh = np.arange(*(h or (0, H)), dtype=np.uint64)
    rw = np.arange(*(w or (0, W)), dtype=np.uint64)
    with np.errstate(over="ignore"):
        idx = (((rn[:, None, None, None] * np.uint64(C) + rc[None, :, None, None]) * np.uint64(H)
                + rh[None, None, :, None]) * np.uint64(W) + rw[None, None, None, :])
    v = _values(hash_index(seed, tensor_id, idx), kind)
    return v * scale if scale != 1.0 else v


def gen_x(N, C, H, W, seed=SEED, kind="act", **block):
    return gen_block((N, C, H, W), seed, TID_X, kind, **block)


def gen_dy(N, F, Ho, Wo, seed=SEED, kind="act", **block):
    return gen_block((N, F, Ho, Wo), seed, TID_DY, kind, **block)


def gen_w(F, C, K, seed=SEED, kind="act"):
    """Weights F x C x K x K (the paper's layout)."""
    s = weight_scale(C, K)
    return gen_block((F, C, K, K), seed, TID_W, kind, scale=s)


# ----------------------------------------------------------------------------
# The same counter-based generator as torch ops (any device): the bench builds
# its resident inputs on the GPU with it instead of hashing gigabytes on the
# host. uint64 arithmetic is emulated in int64 (multiplication wraps mod 2^64;
# right shifts are made logical by masking). Bitwise equal to gen_block
# (tests/test_oracle.py::test_datagen_torch_matches_numpy).
# ----------------------------------------------------------------------------
def _s64(v: int) -> int:
    v &= 0xFFFFFFFFFFFFFFFF
    return v - (1 << 64) if v >= 1 << 63 else v


def _srl(z, s: int):
    import torch
    return torch.bitwise_and(torch.bitwise_right_shift(z, s), (1 << (64 - s)) - 1)


def _splitmix64_t(z):
    z = z + _s64(0x9E3779B97F4A7C15)
    z = torch_xor(z, _srl(z, 30)) * _s64(0xBF58476D1CE4E5B9)
    z = torch_xor(z, _srl(z, 27)) * _s64(0x94D049BB133111EB)
    return torch_xor(z, _srl(z, 31))


def torch_xor(a, b):
    import torch
    return torch.bitwise_xor(a, b)


def gen_block_nhwc_torch(shape, seed: int, tensor_id: int, kind: str = "act", n=None, c=None, h=None,
                         w=None, scale: float = 1.0, c_pad: int | None = None, dtype=None, device="cpu"):
    """gen_block's values of the block, laid out NHWC (channels padded with
    zeros to c_pad), generated with torch ops on `device`, one sample at a
    time; returned in `dtype` (default float64)."""
    import torch
    N, C, H, W = shape
    (n0, n1), (c0, c1), (h0, h1), (w0, w1) = (n or (0, N)), (c or (0, C)), (h or (0, H)), (w or (0, W))
    cp = c_pad if c_pad is not None else c1 - c0
    out = torch.zeros((n1 - n0, h1 - h0, w1 - w0, cp), dtype=dtype or torch.float64, device=device)
    key = int(_key(seed, tensor_id))
    i64 = dict(dtype=torch.int64, device=device)
    rc, rh, rw = torch.arange(c0, c1, **i64), torch.arange(h0, h1, **i64), torch.arange(w0, w1, **i64)
    for k, nn in enumerate(range(n0, n1)):
        idx = ((nn * C + rc[None, None, :]) * H + rh[:, None, None]) * W + rw[None, :, None]  # [h][w][c]
        hv = _splitmix64_t(idx + _s64(key))
        if kind in ("act", "weight"):
            v = torch.bitwise_and(hv, 255).to(torch.float64) / 128.0 - 1.0
        elif kind == "act24":
            v = _srl(hv, 40).to(torch.float64) / float(1 << 23) - 1.0
        else:
            raise ValueError(f"unknown kind {kind!r}")
        if scale != 1.0:
            v = v * scale
        out[k, :, :, :c1 - c0] = v.to(out.dtype)
    return out
