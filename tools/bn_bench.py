"""BN apply / backward microbenchmark through the C ABI (1 GPU): times
dc_bn_apply and dc_bn_backward on one layer's output with CUDA events (after
warm-up), prints achieved GB/s of the algorithmic traffic; small enough to
run under ncu.

usage: python tools/bn_bench.py N F H W [--iters 20]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("shape", type=int, nargs=4)
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    import torch
    import paper_1903_06681_b200 as dc
    N, F, H, W = a.shape
    plan = dc.dc_plan_create(N, F, H, W, F, 3, 1, 1, (1, 1, 1), dc.DC_BF16, None)
    yd, dyd = dc.dc_plan_query(plan, dc.DC_Y), dc.dc_plan_query(plan, dc.DC_DY)
    xd = dc.dc_plan_query(plan, dc.DC_X)
    xb = dc.dc_buffer_alloc(plan, dc.DC_X)
    dyb = dc.dc_buffer_alloc(plan, dc.DC_DY)
    y = (torch.randn((N, H, W, yd["c_pad"]), device="cuda")).to(torch.bfloat16)
    dout = (torch.randn((N, H, W, yd["c_pad"]), device="cuda")).to(torch.bfloat16)
    mean = torch.zeros(F, dtype=torch.float64, device="cuda")
    var = torch.zeros(F, dtype=torch.float64, device="cuda")
    g = torch.ones(F, device="cuda")
    b = torch.zeros(F, device="cuda")
    dg, db = torch.empty_like(g), torch.empty_like(b)
    dc.dc_bn_spatial_stats(plan, y, mean, var, 0)
    by = N * H * W * yd["c_pad"] * 2
    ops = {"stats": (lambda: dc.dc_bn_spatial_stats(plan, y, mean, var, 0), by),
           "apply": (lambda: dc.dc_bn_apply(plan, y, mean, var, g, b, 1e-5, None, dc.DC_RELU, plan, xb), 2 * by),
           "backward": (lambda: dc.dc_bn_backward(plan, dout, y, mean, var, g, b, dyb, 1e-5, None, dc.DC_RELU, dg, db),
                        5 * by)}
    for name, (f, nbytes) in ops.items():
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.iters
        print(f"{name} [{N}, {F}, {H}, {W}]: {ms * 1e3:8.1f} us  {nbytes / (ms * 1e-3) / 1e9:7.0f} GB/s (algorithmic)")
    dc.dc_plan_destroy(plan)
    del xd


if __name__ == "__main__":
    main()
