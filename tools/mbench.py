"""Multi-GPU per-op breakdown of one layer through the C ABI (run under
torchrun, one rank per GPU): halo exchange (P2P / NCCL), forward with and
without the overlapped exchange, backward-filter with and without the dW
allreduce, backward-data, and the fused dc_conv_bwd. Device times with CUDA
events, max over ranks.

usage: torchrun --nproc-per-node 2 tools/mbench.py N C H W F K S P --grid 1,2,1
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("shape", type=int, nargs=8)
    ap.add_argument("--grid", default="auto")
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    import torch
    import torch.distributed as dist
    import paper_1903_06681_b200 as dc
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    uid = [dc.dc_comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = dc.dc_comm_create(rank, world, uid[0], local)
    N, C, H, W, F, K, S, P = a.shape
    grid = (0, 0, 0) if a.grid == "auto" else tuple(int(v) for v in a.grid.split(","))
    plan = dc.dc_plan_create(N, C, H, W, F, K, S, P, grid, dc.DC_BF16, comm)
    chosen, pred = dc.dc_plan_decomp(plan)
    q = {t: dc.dc_plan_query(plan, t) for t in (dc.DC_X, dc.DC_Y, dc.DC_DY, dc.DC_DX)}
    xd, yd, dyd, dxd = q[dc.DC_X], q[dc.DC_Y], q[dc.DC_DY], q[dc.DC_DX]
    xb = dc.wrap_device_buffer(dc.dc_buffer_alloc(plan, dc.DC_X), (xd["n"], xd["hb"], xd["wb"], xd["c_pad"]))
    dyb = dc.wrap_device_buffer(dc.dc_buffer_alloc(plan, dc.DC_DY), (dyd["n"], dyd["hb"], dyd["wb"], dyd["c_pad"]))
    xb.normal_().mul_(0.5)
    dyb.normal_().mul_(0.5)
    xb[..., C:] = 0
    dyb[..., F:] = 0
    w = (torch.randn(F, K, K, xd["c_pad"], device="cuda") * 0.05).to(torch.bfloat16)
    w[..., C:] = 0
    y = torch.empty((yd["n"], yd["h"], yd["w"], yd["c_pad"]), dtype=torch.bfloat16, device="cuda")
    dx = torch.empty((dxd["n"], dxd["h"], dxd["w"], dxd["c_pad"]), dtype=torch.bfloat16, device="cuda")
    dw = torch.empty(F, K, K, C, device="cuda")
    st = torch.cuda.current_stream()
    X, DY = xb.data_ptr(), dyb.data_ptr()
    ops = {
        "halo_x_p2p": lambda: dc.dc_halo_exchange(plan, dc.DC_X, X, 0),
        "halo_x_nccl": lambda: dc.dc_halo_exchange(plan, dc.DC_X, X, dc.DC_HALO_NCCL),
        "halo_dy_p2p": lambda: dc.dc_halo_exchange(plan, dc.DC_DY, DY, 0),
        "fwd_noexch": lambda: dc.dc_conv_fwd(plan, X, w, y, 0),
        "fwd_exch_p2p": lambda: dc.dc_conv_fwd(plan, X, w, y, dc.DC_EXCHANGE),
        "fwd_exch_nccl": lambda: dc.dc_conv_fwd(plan, X, w, y, dc.DC_EXCHANGE | dc.DC_HALO_NCCL),
        "bpw_local": lambda: dc.dc_conv_bwd_filter(plan, X, DY, dw, 0),
        "bpw_allreduce": lambda: dc.dc_conv_bwd_filter(plan, X, DY, dw, dc.DC_ALLREDUCE),
        "bpx_noexch": lambda: dc.dc_conv_bwd_data(plan, DY, w, dx, 0),
        "bpx_exch": lambda: dc.dc_conv_bwd_data(plan, DY, w, dx, dc.DC_EXCHANGE),
        "bwd_fused": lambda: dc.dc_conv_bwd(plan, X, DY, w, dx, dw, dc.DC_DEFAULT_FLAGS),
        "step": lambda: (dc.dc_conv_fwd(plan, X, w, y, dc.DC_EXCHANGE),
                         dc.dc_conv_bwd(plan, X, DY, w, dx, dw, dc.DC_DEFAULT_FLAGS)),
        "step_noexch": lambda: (dc.dc_conv_fwd(plan, X, w, y, 0),
                                dc.dc_conv_bwd(plan, X, DY, w, dx, dw, dc.DC_ALLREDUCE)),
    }
    res = {}
    for name, f in ops.items():
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(a.iters):
            f()
        e1.record(st)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) * 1e3 / a.iters], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res[name] = float(t)
    if rank == 0:
        print(f"shape {a.shape} grid {chosen} (model {pred * 1e6:.1f} us): " +
              "  ".join(f"{k} {v:.1f}" for k, v in res.items()), flush=True)
    dc.dc_plan_destroy(plan)
    dc.dc_comm_destroy(comm)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
