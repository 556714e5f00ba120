"""Redistribution and channel/filter-parallel microbenchmarks over NVLink, one
process per GPU:

  torchrun --nproc-per-node P tools/redist_bench.py [--out FILE]

(1) dc_redistribute of a layer's output between two grids:
    time per call (CUDA events, 20 calls after warm-up, max over ranks), the
    bytes each rank sends to other ranks and the achieved GB/s per GPU, for the
    one-kernel P2P all-to-all and the NCCL send/recv baseline.
(2) A channel/filter-parallel layer (dc_cconv_*) next to the
    same layer on the pure spatial grid (1, P, 1) and on the sample grid: fwd,
    bwd-data and bwd-filter times (the deep 32^2 / 64^2 512-channel layers of
    the 2K mesh model, where spatial shards stop filling the GPU).
Rank 0 prints one JSON line per case."""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1903_06681_b200 as dc  # noqa: E402

REDIST = [  # (name, N, C, H, W, grid from, grid to) of an activation N x C x H x W
    ("conv2_x act", 8, 128, 512, 512, "sample", "spatial"),
    ("conv4_x act", 8, 512, 128, 128, "sample", "spatial"),
    ("conv6_x act", 8, 512, 32, 32, "spatial", "sample"),
]
CF = [("conv6_2", 8, 512, 32, 32, 512, 3, 1, 1), ("conv5_2", 8, 512, 64, 64, 512, 3, 1, 1),
      ("conv4_2", 8, 512, 128, 128, 512, 3, 1, 1)]


def timed(fn, stream, reps=20, warm=3):
    with torch.cuda.stream(stream):
        for _ in range(warm):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / reps], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t[0])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    uid = [dc.dc_comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = dc.dc_comm_create(rank, world, uid[0], local)
    s = torch.cuda.Stream()
    out = open(a.out, "w") if (a.out and rank == 0) else None

    def emit(d):
        if rank == 0:
            print(json.dumps(d), flush=True)
            if out:
                out.write(json.dumps(d) + "\n")

    grids = {"sample": (world, 1, 1), "spatial": (1, world, 1)}
    for name, N, C, H, W, ga, gb in REDIST:
        # the activation is the y of a 3x3/1 layer on grid ga and the x of one on grid gb
        pa = dc.dc_plan_create(N, 16, H, W, C, 3, 1, 1, grids[ga], dc.DC_BF16, comm)
        pb = dc.dc_plan_create(N, C, H, W, 16, 3, 1, 1, grids[gb], dc.DC_BF16, comm)
        qy, qx = dc.dc_plan_query(pa, dc.DC_Y), dc.dc_plan_query(pb, dc.DC_X)
        y = torch.zeros((qy["n"], qy["h"], qy["w"], qy["c_pad"]), dtype=torch.bfloat16, device="cuda")
        xb = dc.dc_buffer_alloc(pb, dc.DC_X)
        r = dc.dc_redist_create(pa, dc.DC_Y, pb, dc.DC_X)
        snd, _ = dc.dc_redist_bytes(r, world)
        moved = sum(v for q, v in enumerate(snd) if q != rank)
        mx = torch.tensor([float(moved)], dtype=torch.float64, device="cuda")
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        for label, flags in (("p2p", 0), ("nccl", dc.DC_HALO_NCCL)):
            ms = timed(lambda: dc.dc_redistribute(r, y, xb, flags, s), s)
            emit({"bench": "redistribute", "case": name, "from": ga, "to": gb, "world": world, "transport": label,
                  "max_bytes_sent_per_rank": int(mx[0]), "us": round(ms * 1e3, 1),
                  "send_GBps_per_gpu": round(float(mx[0]) / (ms * 1e-3) / 1e9, 1)})
        dc.dc_redist_destroy(r)
        dc.dc_plan_destroy(pb)
        dc.dc_plan_destroy(pa)
    for name, N, C, H, W, F, K, S, P in CF:
        Ho, Wo = (H + 2 * P - K) // S + 1, (W + 2 * P - K) // S + 1
        w = (torch.randn(F, K, K, C, device="cuda") * 0.02).to(torch.bfloat16)
        flops = 2 * N * F * C * K * K * Ho * Wo
        res = {"bench": "layer", "case": name, "world": world, "shape": [N, C, H, W, F, K, S, P]}
        # channel / filter parallel (1, world)
        cp = dc.dc_cplan_create(N, C, H, W, F, K, S, P, 1, world, dc.DC_BF16, comm)
        qx, qy = dc.dc_cplan_query(cp, dc.DC_X), dc.dc_cplan_query(cp, dc.DC_Y)
        x = torch.randn((qx["n"], H, W, qx["c"]), device="cuda").to(torch.bfloat16)
        dy = torch.randn((qy["n"], Ho, Wo, qy["c"]), device="cuda").to(torch.bfloat16)
        y = torch.empty((qy["n"], Ho, Wo, qy["c"]), dtype=torch.bfloat16, device="cuda")
        dx = torch.empty((qx["n"], H, W, qx["c"]), dtype=torch.bfloat16, device="cuda")
        dw = torch.empty((F, K, K, qx["c"]), dtype=torch.float32, device="cuda")
        res["channel"] = {op: round(timed(f, s) * 1e3, 1) for op, f in (
            ("fwd_us", lambda: dc.dc_cconv_fwd(cp, x, w, y, 0, s)),
            ("bwd_data_us", lambda: dc.dc_cconv_bwd_data(cp, dy, w, dx, 0, s)),
            ("bwd_filter_us", lambda: dc.dc_cconv_bwd_filter(cp, x, dy, dw, 0, s)))}
        dc.dc_cplan_destroy(cp)
        for gname, grid in (("spatial", (1, world, 1)), ("sample", (world, 1, 1))):
            try:
                pl = dc.dc_plan_create(N, C, H, W, F, K, S, P, grid, dc.DC_BF16, comm)
            except dc.DCError:
                continue
            qx, qy = dc.dc_plan_query(pl, dc.DC_X), dc.dc_plan_query(pl, dc.DC_DY)
            xb = dc.wrap_device_buffer(dc.dc_buffer_alloc(pl, dc.DC_X), (qx["n"], qx["hb"], qx["wb"], qx["c_pad"]))
            dyb = dc.wrap_device_buffer(dc.dc_buffer_alloc(pl, dc.DC_DY), (qy["n"], qy["hb"], qy["wb"], qy["c_pad"]))
            qyy, qdx = dc.dc_plan_query(pl, dc.DC_Y), dc.dc_plan_query(pl, dc.DC_DX)
            y2 = torch.empty((qyy["n"], qyy["h"], qyy["w"], qyy["c_pad"]), dtype=torch.bfloat16, device="cuda")
            dx2 = torch.empty((qdx["n"], qdx["h"], qdx["w"], qdx["c_pad"]), dtype=torch.bfloat16, device="cuda")
            dw2 = torch.empty((F, K, K, C), dtype=torch.float32, device="cuda")
            res[gname] = {op: round(timed(f, s) * 1e3, 1) for op, f in (
                ("fwd_us", lambda: dc.dc_conv_fwd(pl, xb.data_ptr(), w, y2, dc.DC_EXCHANGE, s)),
                ("bwd_data_us", lambda: dc.dc_conv_bwd_data(pl, dyb.data_ptr(), w, dx2, dc.DC_EXCHANGE, s)),
                ("bwd_filter_us", lambda: dc.dc_conv_bwd_filter(pl, xb.data_ptr(), dyb.data_ptr(), dw2, 0, s)))}
            dc.dc_plan_destroy(pl)
        for k in ("channel", "spatial", "sample"):
            if k in res:
                tot = sum(res[k].values())
                res[k]["tflops_fwd_bwd"] = round(3 * flops / (tot * 1e-6) / 1e12, 1)
        emit(res)
    dc.dc_comm_destroy(comm)
    dist.destroy_process_group()
    if out:
        out.close()


if __name__ == "__main__":
    main()
