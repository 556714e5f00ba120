"""C5 sweep + E7 (BASELINE.json configs[4]; "black
markers"): for conv layers over H = W, C = F, K and N, every valid (pN, pH, pW)
grid of P GPUs is RUN (forward with the x halo exchange, backward with the dy
exchange and the dW allreduce) and timed, next to the performance model's
prediction for that grid and the grid the model picks
(decomp = auto). One process per GPU:

  torchrun --nproc-per-node P tools/c5_sweep.py [--out profiles/r2_c5_e7_<P>gpu.jsonl]

Phase 1 ("empirically measured" local costs): the local
fwd / bwd-data / bwd-filter time of every shard the candidate grids produce
(rank 0's block, the largest) is measured on one GPU with L2 evicted, warm-ups
then the mean of ten, the rows spread over the ranks and all-gathered into the
model's cost table. Phase 2: each (layer, grid) is run distributed: three
warm-up steps, then ten steps timed with CUDA events, the max over ranks.
Rank 0 writes one JSON line per layer and prints a summary table."""
import argparse
import json
import os
import statistics
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1903_06681_b200 as dc  # noqa: E402

# the bench's fitted communication terms
ALPHA, BETA, ALPHA_W, OVERLAP = 13e-6, 1 / 700e9, 6e-6, False


def layers():
    out = []
    for H in (128, 512, 2048):
        for C in (16, 64, 256):
            for K in (1, 3):
                for N in (8,):
                    if N * H * H * C > (1 << 31):
                        continue
                    out.append((f"H{H}_C{C}_K{K}_N{N}", N, C, H, H, C, K, 1, K // 2))
    out.append(("H512_16to64_K3_N8", 8, 16, 512, 512, 64, 3, 1, 1))
    out.append(("H512_64to16_K3_N8", 8, 64, 512, 512, 16, 3, 1, 1))
    return out


def grids(N, P):
    for pn in range(P, 0, -1):
        if P % pn or pn > N:
            continue
        rest = P // pn
        for ph in range(rest, 0, -1):
            if rest % ph == 0:
                yield (pn, ph, rest // ph)


def local_costs(shapes, rank, world, scrub):
    """C, Cx, Cw of rank 0's shard of every (layer, grid): warm-ups, then the
    mean of ten with L2 evicted before each."""
    rows = []
    for k, (N, C, H, W, F, K, S, P, grid) in enumerate(shapes):
        if k % world != rank:
            continue
        plan = dc.dc_plan_create_virtual(N, C, H, W, F, K, S, P, grid, 0)
        q = {t: dc.dc_plan_query(plan, t) for t in (dc.DC_X, dc.DC_Y, dc.DC_DY, dc.DC_DX)}
        xd = q[dc.DC_X]

        def buf(d):
            return (torch.rand((d["n"], d["hb"], d["wb"], d["c_pad"]), device="cuda") - 0.5).to(torch.bfloat16)
        x, dy, y, dx = buf(q[dc.DC_X]), buf(q[dc.DC_DY]), buf(q[dc.DC_Y]), buf(q[dc.DC_DX])
        w = ((torch.rand(F, K, K, xd["c_pad"], device="cuda") - 0.5) * 0.1).to(torch.bfloat16)
        dw = torch.empty(F, K, K, C, device="cuda")
        ops = {"fp": lambda: dc.dc_conv_fwd(plan, x, w, y, 0),
               "bpx": lambda: dc.dc_conv_bwd_data(plan, dy, w, dx, 0),
               "bpw": lambda: dc.dc_conv_bwd_filter(plan, x, dy, dw, 0)}
        for op, f in ops.items():
            for _ in range(3):
                f()
            ts = []
            for _ in range(10):
                scrub.fill_(1)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                f()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) / 1e3)
            rows.append(f"{op},{xd['n']},{C},{xd['h']},{xd['w']},{F},{K},{S},{P},{statistics.mean(ts)}")
        dc.dc_plan_destroy(plan)
        del x, dy, y, dx
    return rows


def run_grid(comm, layer, grid, stream, world):
    """One (layer, grid) run distributed; returns (measured ms per fwd+bwd, predicted ms, grid)."""
    name, N, C, H, W, F, K, S, P = layer
    plan = dc.dc_plan_create(N, C, H, W, F, K, S, P, grid, dc.DC_BF16, comm)
    chosen, pred = dc.dc_plan_decomp(plan)
    q = {t: dc.dc_plan_query(plan, t) for t in (dc.DC_X, dc.DC_Y, dc.DC_DY, dc.DC_DX)}
    xd, dyd = q[dc.DC_X], q[dc.DC_DY]
    xb = dc.wrap_device_buffer(dc.dc_buffer_alloc(plan, dc.DC_X), (xd["n"], xd["hb"], xd["wb"], xd["c_pad"]))
    dyb = dc.wrap_device_buffer(dc.dc_buffer_alloc(plan, dc.DC_DY), (dyd["n"], dyd["hb"], dyd["wb"], dyd["c_pad"]))
    xb.copy_((torch.rand(xb.shape, device="cuda") - 0.5).to(torch.bfloat16))
    dyb.copy_((torch.rand(dyb.shape, device="cuda") - 0.5).to(torch.bfloat16))
    yd, dxd = q[dc.DC_Y], q[dc.DC_DX]
    y = torch.empty((yd["n"], yd["h"], yd["w"], yd["c_pad"]), dtype=torch.bfloat16, device="cuda")
    dx = torch.empty((dxd["n"], dxd["h"], dxd["w"], dxd["c_pad"]), dtype=torch.bfloat16, device="cuda")
    w = ((torch.rand(F, K, K, xd["c_pad"], device="cuda") - 0.5) * 0.1).to(torch.bfloat16)
    dw = torch.empty(F, K, K, C, device="cuda")
    sp = stream.cuda_stream
    flags = dc.DC_EXCHANGE | dc.DC_ALLREDUCE

    def step():
        dc.dc_conv_fwd(plan, xb.data_ptr(), w, y, dc.DC_EXCHANGE, sp)
        dc.dc_conv_bwd(plan, xb.data_ptr(), dyb.data_ptr(), w, dx, dw, flags, sp)

    with torch.cuda.stream(stream):
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(10):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / 10], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dc.dc_plan_destroy(plan)
    return float(t[0]), pred * 1e3, chosen


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
    out = a.out or os.path.join(ROOT, "profiles", f"r2_c5_e7_{world}gpu.jsonl")
    L = layers()
    # ---- phase 1: local costs of every shard the candidates produce ----
    shapes, seen = [], set()
    for (name, N, C, H, W, F, K, S, P) in L:
        for g in list(grids(N, world)) + [(1, 1, 1)]:
            try:
                dc.dc_plan_destroy(dc.dc_plan_create_virtual(N, C, H, W, F, K, S, P, g, 0))
            except dc.DCError:
                continue
            key = (N, C, H, W, F, K, S, P, g)
            if key not in seen:
                seen.add(key)
                shapes.append(key)
    scrub = torch.empty(384 << 20, dtype=torch.uint8, device="cuda")
    rows = local_costs(shapes, rank, world, scrub)
    del scrub
    allrows = [None] * world
    dist.all_gather_object(allrows, rows)
    table = os.path.join(ROOT, "gpurun_out" if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else "/tmp",
                         f"c5_cost_table_{world}gpu.csv")
    if rank == 0:
        with open(table, "w") as fh:
            fh.write("op,n,c,h,w,f,k,s,pad,seconds\n")
            for r in allrows:
                fh.write("\n".join(r) + ("\n" if r else ""))
    dist.barrier()
    dc.dc_model_load_table(table)
    dc.dc_model_set_comm(ALPHA, BETA)
    dc.dc_model_set_strided_latency(ALPHA_W)
    dc.dc_model_set_overlap(OVERLAP)
    # ---- phase 2: every grid run distributed, vs the model ----
    stream = torch.cuda.Stream()
    res = []
    for layer in L:
        name, N, C, H, W, F, K, S, P = layer
        cands = []
        for g in grids(N, world):
            try:
                dc.dc_plan_destroy(dc.dc_plan_create_virtual(N, C, H, W, F, K, S, P, g, 0))
            except dc.DCError:
                continue
            meas, pred, _ = run_grid(comm, layer, g, stream, world)
            cands.append({"grid": list(g), "measured_ms": round(meas, 4), "predicted_ms": round(pred, 4)})
        auto, _ = dc.dc_model_choose(N, C, H, W, F, K, S, P, world)
        best = min(cands, key=lambda c: c["measured_ms"])
        pick = next(c for c in cands if c["grid"] == list(auto))
        r = {"layer": name, "shape_NCHW_F_K_S_P": [N, C, H, W, F, K, S, P], "world": world, "candidates": cands,
             "model_pick": list(auto), "measured_best": best["grid"],
             "pick_vs_best": round(pick["measured_ms"] / best["measured_ms"], 4),
             "pick_pred_err": round(pick["predicted_ms"] / pick["measured_ms"] - 1, 4)}
        res.append(r)
        if rank == 0:
            print(json.dumps(r), flush=True)
    if rank == 0:
        with open(out, "w") as fh:
            for r in res:
                fh.write(json.dumps(r) + "\n")
        hits = sum(1 for r in res if r["model_pick"] == r["measured_best"])
        loss = statistics.mean(r["pick_vs_best"] for r in res)
        err = statistics.median(abs(r["pick_pred_err"]) for r in res)
        print(f"E7 summary ({world} GPUs, {len(res)} layers): model picks the measured best grid in {hits}; "
              f"mean time of the pick / best {loss:.3f}; median |predicted/measured - 1| of the pick {err:.3f}",
              flush=True)
    dc.dc_comm_destroy(comm)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
