"""oracle.network -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The non-convolution layers the paper runs on the same sample / spatial
decomposition, as plain
fp64 NCHW numpy, written from their definitions:

  * batch normalisation with the spatially aggregated statistics of
    PAPER.md:149 (reading R11: mean and biased variance over the samples of
    the group and the whole spatial extent), y_hat = (y - mu) / sqrt(var +
    eps), out = gamma y_hat + beta (reading R27: the standard BN transform;
    the paper gives no formula), then an optional residual add and ReLU
    (ResNet blocks; the mesh network's conv-BN-ReLU stack,
    PAPER.md:236);
  * its backward with the group sums sum(g) and sum(g y_hat) that the spatial
    group must aggregate ("aggregates over the spatial
    distribution");
  * 3x3 / stride-2 max pooling (ResNet's stem), forward and
    backward (the gradient goes to the first maximum of each window in
    (a, b) order).

Every function is the definition written out; no blocking or fusion."""
from __future__ import annotations

import numpy as np


def bn_forward(y, mean, var, gamma, beta, eps: float = 1e-5):
    """out[n,c,i,j] = gamma[c] (y - mean[c]) / sqrt(var[c] + eps) + beta[c]."""
    y = np.asarray(y, dtype=np.float64)
    ch = (None, slice(None), None, None)
    mean = np.asarray(mean, dtype=np.float64)[ch]
    sd = np.sqrt(np.asarray(var, dtype=np.float64) + eps)[ch]
    return np.asarray(gamma, dtype=np.float64)[ch] * (y - mean) / sd + np.asarray(beta, dtype=np.float64)[ch]


def bn_relu_forward(y, mean, var, gamma, beta, eps: float = 1e-5, residual=None, relu: bool = True):
    """out = relu(BN(y) + residual) (residual and relu optional)."""
    z = bn_forward(y, mean, var, gamma, beta, eps)
    if residual is not None:
        z = z + np.asarray(residual, dtype=np.float64)
    return np.maximum(z, 0.0) if relu else z


def bn_relu_backward(dout, y, mean, var, gamma, beta, eps: float = 1e-5, residual=None, relu: bool = True):
    """Gradients of out = relu(BN(y) + residual) with the batch statistics a
    function of y over the whole tensor (the group):
        g       = dout * [BN(y) + residual > 0]        (ReLU mask)
        y_hat   = (y - mean) / sqrt(var + eps)
        dbeta   = sum g,  dgamma = sum g y_hat          (per channel)
        dy      = gamma / sqrt(var + eps) (g - dbeta / M - y_hat dgamma / M),  M = N H W
        dresidual = g.
    Returns (dy, dgamma, dbeta, dresidual)."""
    y = np.asarray(y, dtype=np.float64)
    dout = np.asarray(dout, dtype=np.float64)
    N, C, H, W = y.shape
    M = float(N * H * W)
    mean = np.asarray(mean, dtype=np.float64)[None, :, None, None]
    sd = np.sqrt(np.asarray(var, dtype=np.float64) + eps)[None, :, None, None]
    yhat = (y - mean) / sd
    z = np.asarray(gamma, dtype=np.float64)[None, :, None, None] * yhat + np.asarray(beta, dtype=np.float64)[None, :, None, None]
    if residual is not None:
        z = z + np.asarray(residual, dtype=np.float64)
    g = dout * (z > 0) if relu else dout
    dbeta = g.sum(axis=(0, 2, 3))
    dgamma = (g * yhat).sum(axis=(0, 2, 3))
    dy = np.asarray(gamma, dtype=np.float64)[None, :, None, None] / sd * (
        g - dbeta[None, :, None, None] / M - yhat * dgamma[None, :, None, None] / M)
    return dy, dgamma, dbeta, g


def maxpool_fwd(x, K: int = 3, S: int = 2, P: int = 1):
    """out[n,c,i,j] = max over a, b < K of x[n,c,S i + a - P, S j + b - P]
    (positions outside the input excluded); also the argmax window index a K + b
    (the first maximum in (a, b) order). Returns (out, argmax)."""
    x = np.asarray(x, dtype=np.float64)
    N, C, H, W = x.shape
    Ho, Wo = (H + 2 * P - K) // S + 1, (W + 2 * P - K) // S + 1
    xp = np.full((N, C, H + 2 * P + S, W + 2 * P + S), -np.inf)
    xp[:, :, P:P + H, P:P + W] = x
    out = np.full((N, C, Ho, Wo), -np.inf)
    arg = np.zeros((N, C, Ho, Wo), dtype=np.int64)
    for a in range(K):
        for b in range(K):
            v = xp[:, :, a:a + S * Ho:S, b:b + S * Wo:S][:, :, :Ho, :Wo]
            better = v > out
            out = np.where(better, v, out)
            arg = np.where(better, a * K + b, arg)
    return out, arg


def maxpool_bwd(dout, argmax, H: int, W: int, K: int = 3, S: int = 2, P: int = 1):
    """dx[n,c,u,v] = sum over outputs whose argmax is (u, v) of dout."""
    dout = np.asarray(dout, dtype=np.float64)
    N, C, Ho, Wo = dout.shape
    dx = np.zeros((N, C, H, W))
    for i in range(Ho):
        for j in range(Wo):
            a, b = argmax[:, :, i, j] // K, argmax[:, :, i, j] % K
            u, v = S * i + a - P, S * j + b - P
            for n in range(N):
                for c in range(C):
                    dx[n, c, u[n, c], v[n, c]] += dout[n, c, i, j]
    return dx
