"""Per-layer kernel microbenchmark through the C ABI (1 GPU): times fwd,
bwd-filter and bwd-data of one layer with CUDA events (after warm-up) and
prints achieved TFLOP/s; small enough to run under ncu.

usage: python tools/kbench.py N C H W F K S P [--iters 20] [--ops fwd,bpw,bpx]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("shape", type=int, nargs=8)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--ops", default="fwd,bpw,bpx")
    ap.add_argument("--bn-fused", action="store_true", help="forward with DC_BN_STATS (as bench.py runs it)")
    ap.add_argument("--flush", action="store_true",
                    help="evict L2 before every timed op (cold inputs, like the bench step)")
    a = ap.parse_args()
    import torch
    from paper_1903_06681_b200 import build
    build.build()
    import paper_1903_06681_b200 as dc
    N, C, H, W, F, K, S, P = a.shape
    plan = dc.dc_plan_create(N, C, H, W, F, K, S, P, (1, 1, 1), dc.DC_BF16, None)
    q = {t: dc.dc_plan_query(plan, t) for t in (dc.DC_X, dc.DC_Y, dc.DC_DY, dc.DC_DX)}
    g = torch.Generator(device="cuda").manual_seed(1903)

    def buf(d):
        t = (torch.randint(-128, 128, (d["n"], d["hb"], d["wb"], d["c_pad"]), generator=g, device="cuda")
             .to(torch.bfloat16) / 128)
        t[..., d["c"]:] = 0
        return t
    x, dy = buf(q[dc.DC_X]), buf(q[dc.DC_DY])
    y, dx = torch.empty_like(buf(q[dc.DC_Y])), torch.empty_like(buf(q[dc.DC_DX]))
    w = torch.randn(F, K, K, q[dc.DC_X]["c_pad"], device="cuda").to(torch.bfloat16) * 0.05
    w[..., C:] = 0
    dw = torch.empty(F, K, K, C, device="cuda")
    Ho, Wo = (H + 2 * P - K) // S + 1, (W + 2 * P - K) // S + 1
    flops = 2.0 * N * F * C * K * K * Ho * Wo
    fwd_flags = dc.DC_BN_STATS if a.bn_fused else 0
    ops = {"fwd": lambda: dc.dc_conv_fwd(plan, x, w, y, fwd_flags),
           "bpw": lambda: dc.dc_conv_bwd_filter(plan, x, dy, dw, 0),
           "bpx": lambda: dc.dc_conv_bwd_data(plan, dy, w, dx, 0),
           "bn": lambda: dc.dc_bn_spatial_stats(plan, y, mean, var, dc.DC_BN_LOCAL | (dc.DC_BN_FROM_FWD if a.bn_fused else 0), 0)}
    mean = torch.empty(F, dtype=torch.float64, device="cuda")
    var = torch.empty(F, dtype=torch.float64, device="cuda")
    for name in a.ops.split(","):
        f = ops[name]
        for _ in range(a.warmup):
            f()
        torch.cuda.synchronize()
        if a.flush:
            scrub = torch.empty(384 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(a.iters)]
            for e0, e1 in ev:
                scrub.fill_(1)
                e0.record()
                f()
                e1.record()
            torch.cuda.synchronize()
            us = sum(e0.elapsed_time(e1) for e0, e1 in ev) * 1e3 / a.iters
        else:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.iters):
                f()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / a.iters
        if name == "bn":
            print(f"{name} {a.shape}: {us:8.1f} us  {y.numel() * 2 / us / 1e3:7.1f} GB/s", flush=True)
        else:
            print(f"{name} {a.shape}: {us:8.1f} us  {flops / us / 1e6:7.1f} TFLOP/s", flush=True)
    dc.dc_plan_destroy(plan)


if __name__ == "__main__":
    main()
