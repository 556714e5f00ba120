"""Test plumbing: move seeded global NCHW tensors (float64, bf16-exact) into
the library's NHWC shard buffers and back. No convolution arithmetic here."""
from __future__ import annotations

import numpy as np
import torch

import paper_1903_06681_b200 as dc


def fill_buffer(glob: np.ndarray, desc: dict, kind: str = "x", device="cuda") -> torch.Tensor:
    """Margined NHWC bf16 buffer of `desc` holding the global tensor's rows
    [h0-halo_n, h0+h+halo_s) x cols [w0-halo_w, w0+w+halo_e) of samples
    [n0, n0+n) (halo included when with_halo)."""
    n0, n, h0, w0 = desc["n0"], desc["n"], desc["h0"], desc["w0"]
    hb, wb, cp, c = desc["hb"], desc["wb"], desc["c_pad"], desc["c"]
    r0, c0 = h0 - desc["halo_n"], w0 - desc["halo_w"]
    blk = glob[n0:n0 + n, :c, r0:r0 + hb, c0:c0 + wb]            # N C hb wb
    buf = np.zeros((n, hb, wb, cp))
    buf[..., :c] = blk.transpose(0, 2, 3, 1)
    return torch.tensor(buf, dtype=torch.bfloat16, device=device).contiguous()


def fill_owned_only(glob: np.ndarray, desc: dict, device="cuda") -> torch.Tensor:
    """Same buffer with the margins left zero (they must come from the exchange)."""
    t = torch.zeros((desc["n"], desc["hb"], desc["wb"], desc["c_pad"]), dtype=torch.bfloat16, device=device)
    hn, hw = desc["halo_n"], desc["halo_w"]
    own = glob[desc["n0"]:desc["n0"] + desc["n"], :desc["c"], desc["h0"]:desc["h0"] + desc["h"],
               desc["w0"]:desc["w0"] + desc["w"]]
    t[:, hn:hn + desc["h"], hw:hw + desc["w"], :desc["c"]] = torch.tensor(own.transpose(0, 2, 3, 1), dtype=torch.bfloat16)
    return t


def empty_dense(desc: dict, device="cuda") -> torch.Tensor:
    return torch.full((desc["n"], desc["hb"], desc["wb"], desc["c_pad"]), float("nan"),
                      dtype=torch.bfloat16, device=device)


def owned_nchw(t: torch.Tensor, desc: dict) -> np.ndarray:
    """Owned block of an NHWC buffer as float64 NCHW (logical channels only)."""
    hn, hw = desc["halo_n"], desc["halo_w"]
    blk = t[:, hn:hn + desc["h"], hw:hw + desc["w"], :desc["c"]]
    return blk.float().cpu().numpy().astype(np.float64).transpose(0, 3, 1, 2)


def weights_gpu(w: np.ndarray, cp: int, device="cuda") -> torch.Tensor:
    """F x C x K x K (paper layout) -> bf16 [F][K][K][cp]."""
    F, C, K, _ = w.shape
    out = np.zeros((F, K, K, cp))
    out[..., :C] = w.transpose(0, 2, 3, 1)
    return torch.tensor(out, dtype=torch.bfloat16, device=device).contiguous()


def dw_to_fckk(dw: torch.Tensor, C: int) -> np.ndarray:
    """fp32 [F][K][K][cp] -> float64 F x C x K x K."""
    return dw[..., :C].double().cpu().numpy().transpose(0, 3, 1, 2)


def rel_l2(got: np.ndarray, ref: np.ndarray) -> float:
    den = np.linalg.norm(ref.ravel())
    return float(np.linalg.norm((got - ref).ravel()) / (den if den > 0 else 1.0))


def rel_max(got: np.ndarray, ref: np.ndarray) -> float:
    den = np.abs(ref).max()
    return float(np.abs(got - ref).max() / (den if den > 0 else 1.0))


def elementwise_bound(ref: np.ndarray, S: np.ndarray, n_terms: int, k_step: int, out_bf16: bool,
                      extra_adds: int = 32) -> np.ndarray:
    """Per-element error bound of a tensor-core result against the exact value
    (DESIGN.md §7): products of the (exactly representable) inputs are exact
    in fp32; the fp32 accumulation adds one partial per K step of k_step
    terms (16 bf16 / 8 tf32) plus at most `extra_adds` more (the reduction
    inside an MMA, split-K partials), so |acc - exact| <= m 2^-24 S with
    m = n_terms / k_step + extra_adds and S = sum of |terms| (the oracle run
    on absolute values); a bf16 output adds its round-to-nearest error,
    2^-8 |value| (8-bit significand)."""
    m = n_terms / float(k_step) + extra_adds
    acc = m * 2.0 ** -24 * S
    if out_bf16:
        return 2.0 ** -8 * (np.abs(ref) + acc) + acc + 1e-30
    return acc + 1e-30


def assert_elementwise(name: str, got: np.ndarray, ref: np.ndarray, bound: np.ndarray):
    assert np.isfinite(got).all(), f"{name}: non-finite values"
    err = np.abs(got - ref)
    bad = err > bound
    assert not bad.any(), (f"{name}: {int(bad.sum())} of {bad.size} elements over the derived bound "
                           f"(worst {float((err / bound).max()):.2f}x, max err {float(err.max()):.3e})")
