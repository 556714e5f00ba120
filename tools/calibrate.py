"""Measure the local convolution costs C, Cx, Cw of the paper's performance
model ("we use empirically measured ... runtimes") on this
GPU: for every unique layer of the bench workloads and every valid grid at
1/2/4/8 ranks, rank 0's shard (the largest block) is run through the C ABI on
one GPU (virtual plan, no exchange) with L2 evicted before each timed op:
several warm-up runs, then the average of ten, written as a
table row "op,n,c,h,w,f,k,s,pad,seconds" keyed by the local extents the model
looks up (dc_model_load_table).

usage: python tools/calibrate.py [--out profiles/cost_table_b200.csv] [--ranks 1,2,4,8]
"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def grids(N, P):
    for pn in range(P, 0, -1):
        if P % pn or pn > N:
            continue
        rest = P // pn
        for ph in range(rest, 0, -1):
            if rest % ph == 0:
                yield (pn, ph, rest // ph)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "cost_table_b200.csv"))
    ap.add_argument("--ranks", default="1,2,4,8")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workloads", default="mesh2k,resnet_layers")
    a = ap.parse_args()
    import torch
    from paper_1903_06681_b200 import build
    build.build()
    import paper_1903_06681_b200 as dc
    import bench
    shapes = []
    for wl in a.workloads.split(","):
        for l in bench.WORKLOADS[wl]:
            if tuple(l[1:]) not in shapes:
                shapes.append(tuple(l[1:]))
    scrub = torch.empty(384 << 20, dtype=torch.uint8, device="cuda")
    rows, seen = [], set()
    for (N, C, H, W, F, K, S, P) in shapes:
        for Pn in (int(v) for v in a.ranks.split(",")):
            for grid in grids(N, Pn):
                try:
                    plan = dc.dc_plan_create_virtual(N, C, H, W, F, K, S, P, grid, 0)
                except dc.DCError:
                    continue  # invalid partition of this layer
                q = {t: dc.dc_plan_query(plan, t) for t in (dc.DC_X, dc.DC_Y, dc.DC_DY, dc.DC_DX)}
                xd = q[dc.DC_X]
                key = (xd["n"], C, xd["h"], xd["w"], F, K, S, P)
                if key in seen:
                    dc.dc_plan_destroy(plan)
                    continue
                seen.add(key)

                def buf(d, dt=torch.bfloat16):
                    return (torch.rand((d["n"], d["hb"], d["wb"], d["c_pad"]), device="cuda") - 0.5).to(dt)
                x, dy = buf(q[dc.DC_X]), buf(q[dc.DC_DY])
                y, dx = buf(q[dc.DC_Y]), buf(q[dc.DC_DX])
                w = ((torch.rand(F, K, K, xd["c_pad"], device="cuda") - 0.5) * 0.1).to(torch.bfloat16)
                dw = torch.empty(F, K, K, C, device="cuda")
                ops = {"fp": lambda: dc.dc_conv_fwd(plan, x, w, y, 0),
                       "bpx": lambda: dc.dc_conv_bwd_data(plan, dy, w, dx, 0),
                       "bpw": lambda: dc.dc_conv_bwd_filter(plan, x, dy, dw, 0)}
                for op, f in ops.items():
                    for _ in range(a.warmup):
                        f()
                    torch.cuda.synchronize()
                    ts = []
                    for _ in range(a.iters):
                        scrub.fill_(1)
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record()
                        f()
                        e1.record()
                        torch.cuda.synchronize()
                        ts.append(e0.elapsed_time(e1) / 1e3)
                    rows.append((op,) + key + (statistics.mean(ts),))
                dc.dc_plan_destroy(plan)
                print(f"{(N, C, H, W, F, K, S, P)} grid {grid}: local {key[:4]} "
                      + " ".join(f"{r[0]} {r[-1] * 1e6:.1f}us" for r in rows[-3:]), flush=True)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as fh:
        fh.write("op,n,c,h,w,f,k,s,pad,seconds\n")
        for r in rows:
            fh.write(",".join(str(v) for v in r) + "\n")
    print(f"wrote {len(rows)} rows to {a.out}")


if __name__ == "__main__":
    main()
