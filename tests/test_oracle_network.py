"""Pins of oracle/network.py (the NEXT-1 layers: spatial BN apply / backward
with ReLU and residual, max pooling) against what mathematics and a library
special case fix -- never against the oracle's own formulas:
  * closed forms: normalised output has per-channel mean 0 and variance
    var / (var + eps) when gamma = 1, beta = 0; max pooling of a constant;
  * library special cases: torch CPU fp64 batch_norm (training statistics) +
    relu and max_pool2d, and their autograd gradients;
  * central finite differences of the scalar <dout, out(y)> (statistics
    recomputed from y, as the group does);
  * the spatial-group invariant: the backward's group sums are the sums of
    per-shard sums over any spatial partition."""
import numpy as np
import torch
import torch.nn.functional as Fn

import oracle
from oracle import network as net
from oracle import partition as part

rng = np.random.default_rng(27)


def _stats(y):
    return oracle.bn_stats(y)


def test_bn_forward_closed_form():
    y = rng.standard_normal((3, 5, 7, 6)) * 3 + 2
    m, v = _stats(y)
    out = net.bn_forward(y, m, v, np.ones(5), np.zeros(5), eps=1e-5)
    np.testing.assert_allclose(out.mean(axis=(0, 2, 3)), 0, atol=1e-12)
    np.testing.assert_allclose(out.var(axis=(0, 2, 3)), v / (v + 1e-5), rtol=1e-12)
    g, b = rng.standard_normal(5), rng.standard_normal(5)
    out2 = net.bn_forward(y, m, v, g, b, eps=1e-5)
    np.testing.assert_allclose(out2, g[None, :, None, None] * out + b[None, :, None, None], rtol=1e-12, atol=1e-12)


def test_bn_relu_forward_vs_torch():
    y = rng.standard_normal((2, 4, 5, 6))
    res = rng.standard_normal((2, 4, 5, 6))
    g, b = rng.standard_normal(4), rng.standard_normal(4)
    m, v = _stats(y)
    ref = torch.relu(Fn.batch_norm(torch.tensor(y), None, None, torch.tensor(g), torch.tensor(b), training=True,
                                   eps=1e-5) + torch.tensor(res)).numpy()
    np.testing.assert_allclose(net.bn_relu_forward(y, m, v, g, b, 1e-5, residual=res), ref, rtol=1e-11, atol=1e-12)


def test_bn_relu_backward_vs_autograd_and_fd():
    y = rng.standard_normal((2, 3, 4, 5))
    res = rng.standard_normal((2, 3, 4, 5)) * 0.5
    g, b = rng.standard_normal(3), rng.standard_normal(3)
    dout = rng.standard_normal((2, 3, 4, 5))
    m, v = _stats(y)
    dy, dgam, dbet, dres = net.bn_relu_backward(dout, y, m, v, g, b, 1e-5, residual=res)
    ty, tg, tb, tr = (torch.tensor(a, requires_grad=True) for a in (y, g, b, res))
    out = torch.relu(Fn.batch_norm(ty, None, None, tg, tb, training=True, eps=1e-5) + tr)
    (out * torch.tensor(dout)).sum().backward()
    np.testing.assert_allclose(dy, ty.grad.numpy(), rtol=1e-9, atol=1e-11)
    np.testing.assert_allclose(dgam, tg.grad.numpy(), rtol=1e-9, atol=1e-11)
    np.testing.assert_allclose(dbet, tb.grad.numpy(), rtol=1e-9, atol=1e-11)
    np.testing.assert_allclose(dres, tr.grad.numpy(), rtol=1e-9, atol=1e-11)

    def L(yy):  # statistics recomputed from the perturbed input
        mm, vv = _stats(yy)
        return float((dout * net.bn_relu_forward(yy, mm, vv, g, b, 1e-5, residual=res)).sum())
    h = 1e-6
    for idx in [(0, 0, 0, 0), (1, 2, 3, 4), (0, 1, 2, 1)]:
        yp, ym = y.copy(), y.copy()
        yp[idx] += h
        ym[idx] -= h
        fd = (L(yp) - L(ym)) / (2 * h)
        assert abs(fd - dy[idx]) <= 1e-6 * max(1.0, abs(fd)), (idx, fd, dy[idx])


def test_bn_backward_group_sums_are_partition_sums():
    """the backward's per-channel sums over the group equal the
    sums of the per-shard sums of any spatial partition."""
    y = rng.standard_normal((2, 3, 9, 7))
    dout = rng.standard_normal((2, 3, 9, 7))
    g, b = rng.standard_normal(3), rng.standard_normal(3)
    m, v = _stats(y)
    _, dgam, dbet, gmask = net.bn_relu_backward(dout, y, m, v, g, b)
    yhat = (y - m[None, :, None, None]) / np.sqrt(v + 1e-5)[None, :, None, None]
    for ph, pw in [(2, 1), (3, 2)]:
        sg, sgy = np.zeros(3), np.zeros(3)
        for ih in range(ph):
            for iw in range(pw):
                h0, h1 = part.blocked(9, ph, ih)
                w0, w1 = part.blocked(7, pw, iw)
                sg += gmask[:, :, h0:h1, w0:w1].sum(axis=(0, 2, 3))
                sgy += (gmask * yhat)[:, :, h0:h1, w0:w1].sum(axis=(0, 2, 3))
        np.testing.assert_allclose(sg, dbet, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(sgy, dgam, rtol=1e-12, atol=1e-12)


def test_maxpool_vs_torch_and_constant():
    x = rng.permutation(2 * 3 * 11 * 10).reshape(2, 3, 11, 10).astype(np.float64)  # distinct values
    out, arg = net.maxpool_fwd(x, 3, 2, 1)
    tx = torch.tensor(x, requires_grad=True)
    ref = Fn.max_pool2d(tx, 3, 2, 1)
    np.testing.assert_array_equal(out, ref.detach().numpy())
    dout = rng.standard_normal(out.shape)
    (ref * torch.tensor(dout)).sum().backward()
    np.testing.assert_allclose(net.maxpool_bwd(dout, arg, 11, 10, 3, 2, 1), tx.grad.numpy(), rtol=0, atol=1e-12)
    c, _ = net.maxpool_fwd(np.full((1, 1, 8, 8), 2.5))
    assert (c == 2.5).all() and c.shape == (1, 1, 4, 4)
