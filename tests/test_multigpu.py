"""Multi-GPU parity (one process per GPU, NCCL + CUDA-IPC P2P), run under
`gpurun --gpus 2|4`:
  * halo exchange is bit-exact (P2P stores and the NCCL send/recv baseline);
  * partitioned y and dx are BITWISE equal to the 1-GPU result of the same
    kernel computed on the same device (north_star);
  * the allreduced dW matches the 1-GPU dW within the fp32 bar (1e-4,
    different summation tree, reading R10);
  * spatially aggregated BN statistics match the 1-GPU statistics within the
    derived fp32-group bound."""
import os
import socket
import traceback

import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

CASES = {
    2: [((2, 16, 24, 20, 32, 3, 1, 1), (1, 2, 1)), ((2, 16, 24, 20, 32, 3, 1, 1), (1, 1, 2)),
        ((2, 16, 24, 20, 32, 3, 1, 1), (2, 1, 1)), ((1, 3, 40, 36, 64, 7, 2, 3), (1, 2, 1)),
        ((2, 64, 16, 16, 64, 3, 1, 1), (1, 2, 1)), ((1, 18, 33, 35, 64, 3, 2, 1), (1, 1, 2))],
    4: [((2, 16, 24, 20, 32, 3, 1, 1), (1, 2, 2)), ((2, 16, 24, 20, 32, 3, 1, 1), (2, 2, 1)),
        ((1, 32, 40, 24, 48, 5, 1, 2), (1, 4, 1)), ((1, 3, 40, 36, 64, 7, 2, 3), (1, 2, 2))],
}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, errq, env=None):
    try:
        os.environ.update(env or {})
        import sys
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, root)
        import torch.distributed as dist
        import datagen
        import paper_1903_06681_b200 as dc
        from tests.gpu_util import fill_buffer, fill_owned_only, weights_gpu, dw_to_fckk, rel_max
        torch.cuda.set_device(rank)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        uid = [dc.dc_comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = dc.dc_comm_create(rank, world, uid[0], rank)
        for shape, grid in CASES[world]:
            N, C, H, W, F, K, S, P = shape
            Ho, Wo = (H + 2 * P - K) // S + 1, (W + 2 * P - K) // S + 1
            x, w, dy = datagen.gen_x(N, C, H, W), datagen.gen_w(F, C, K), datagen.gen_dy(N, F, Ho, Wo)
            # 1-GPU reference of the same kernels on this device
            ref = dc.dc_plan_create(N, C, H, W, F, K, S, P, (1, 1, 1), dc.DC_BF16, None)
            rx, ry = dc.dc_plan_query(ref, dc.DC_X), dc.dc_plan_query(ref, dc.DC_Y)
            rdy, rdx = dc.dc_plan_query(ref, dc.DC_DY), dc.dc_plan_query(ref, dc.DC_DX)
            wb = weights_gpu(w, rx["c_pad"])
            Y = torch.empty((ry["n"], ry["h"], ry["w"], ry["c_pad"]), dtype=torch.bfloat16, device="cuda")
            DX = torch.empty((rdx["n"], rdx["h"], rdx["w"], rdx["c_pad"]), dtype=torch.bfloat16, device="cuda")
            DW = torch.empty((F, K, K, C), dtype=torch.float32, device="cuda")
            xr, dyr = fill_buffer(x, rx), fill_buffer(dy, rdy)
            dc.dc_conv_fwd(ref, xr, wb, Y, 0)
            dc.dc_conv_bwd_data(ref, dyr, wb, DX, 0)
            dc.dc_conv_bwd_filter(ref, xr, dyr, DW, 0)
            mean_r = torch.zeros(F, dtype=torch.float64, device="cuda")
            var_r = torch.zeros(F, dtype=torch.float64, device="cuda")
            dc.dc_bn_spatial_stats(ref, Y, mean_r, var_r, True)
            torch.cuda.synchronize()
            # distributed plan
            plan = dc.dc_plan_create(N, C, H, W, F, K, S, P, grid, dc.DC_BF16, comm)
            xd, yd = dc.dc_plan_query(plan, dc.DC_X), dc.dc_plan_query(plan, dc.DC_Y)
            dyd, dxd = dc.dc_plan_query(plan, dc.DC_DY), dc.dc_plan_query(plan, dc.DC_DX)
            xb = dc.wrap_device_buffer(dc.dc_buffer_alloc(plan, dc.DC_X), (xd["n"], xd["hb"], xd["wb"], xd["c_pad"]))
            dyb = dc.wrap_device_buffer(dc.dc_buffer_alloc(plan, dc.DC_DY), (dyd["n"], dyd["hb"], dyd["wb"], dyd["c_pad"]))
            full_x, full_dy = fill_buffer(x, xd), fill_buffer(dy, dyd)
            tag = f"rank {rank} shape {shape} grid {grid}"
            # (1) halo exchange bit-exact: NCCL baseline, then direct P2P
            for flags in (dc.DC_HALO_NCCL, 0):
                xb.copy_(fill_owned_only(x, xd))
                torch.cuda.synchronize()
                dist.barrier()
                dc.dc_halo_exchange(plan, dc.DC_X, xb, flags)
                torch.cuda.synchronize()
                assert torch.equal(xb, full_x), f"{tag}: x halo (flags {flags}) not bit-exact"
            # (2) forward with the overlapped exchange; y bitwise == 1-GPU
            xb.copy_(fill_owned_only(x, xd))
            y = torch.empty((yd["n"], yd["h"], yd["w"], yd["c_pad"]), dtype=torch.bfloat16, device="cuda")
            torch.cuda.synchronize()
            dist.barrier()
            dc.dc_conv_fwd(plan, xb.data_ptr(), wb, y, dc.DC_EXCHANGE | dc.DC_FORCE_OVERLAP)
            torch.cuda.synchronize()
            ys = Y[yd["n0"]:yd["n0"] + yd["n"], yd["h0"]:yd["h0"] + yd["h"], yd["w0"]:yd["w0"] + yd["w"]]
            assert torch.equal(y, ys), f"{tag}: y not bitwise equal to 1-GPU"
            # (2b) the non-overlapped schedule (exchange, then one pass): same bits
            xb.copy_(fill_owned_only(x, xd))
            y.zero_()
            torch.cuda.synchronize()
            dist.barrier()
            dc.dc_conv_fwd(plan, xb.data_ptr(), wb, y, dc.DC_EXCHANGE | dc.DC_NO_OVERLAP)
            torch.cuda.synchronize()
            assert torch.equal(y, ys), f"{tag}: y (DC_NO_OVERLAP) not bitwise equal to 1-GPU"
            dyb.copy_(fill_owned_only(dy, dyd))
            dx = torch.empty((dxd["n"], dxd["h"], dxd["w"], dxd["c_pad"]), dtype=torch.bfloat16, device="cuda")
            torch.cuda.synchronize()
            dist.barrier()
            dc.dc_conv_bwd_data(plan, dyb.data_ptr(), wb, dx, dc.DC_EXCHANGE | dc.DC_NO_OVERLAP)
            torch.cuda.synchronize()
            dxs = DX[dxd["n0"]:dxd["n0"] + dxd["n"], dxd["h0"]:dxd["h0"] + dxd["h"], dxd["w0"]:dxd["w0"] + dxd["w"]]
            assert torch.equal(dx, dxs), f"{tag}: dx (DC_NO_OVERLAP) not bitwise equal to 1-GPU"
            # (3) backward with dy exchange || wgrad, allreduce || dgrad
            dyb.copy_(fill_owned_only(dy, dyd))
            dx = torch.empty((dxd["n"], dxd["h"], dxd["w"], dxd["c_pad"]), dtype=torch.bfloat16, device="cuda")
            dw = torch.empty((F, K, K, C), dtype=torch.float32, device="cuda")
            torch.cuda.synchronize()
            dist.barrier()
            dc.dc_conv_bwd(plan, xb.data_ptr(), dyb.data_ptr(), wb, dx, dw, dc.DC_DEFAULT_FLAGS)
            torch.cuda.synchronize()
            assert torch.equal(dyb, full_dy), f"{tag}: dy halo not bit-exact"
            dxs = DX[dxd["n0"]:dxd["n0"] + dxd["n"], dxd["h0"]:dxd["h0"] + dxd["h"], dxd["w0"]:dxd["w0"] + dxd["w"]]
            assert torch.equal(dx, dxs), f"{tag}: dx not bitwise equal to 1-GPU"
            e = rel_max(dw_to_fckk(dw, C), dw_to_fckk(DW, C))
            assert e <= 1e-4, f"{tag}: dW rel err {e}"
            # (4) spatial BN statistics over the ranks sharing the samples
            mean = torch.zeros(F, dtype=torch.float64, device="cuda")
            var = torch.zeros(F, dtype=torch.float64, device="cuda")
            dc.dc_bn_spatial_stats(plan, y, mean, var, False)
            torch.cuda.synchronize()
            if grid[0] == 1:  # group = all ranks = the whole batch
                # both sides: fp32 groups of 8 then fp64, different groupings
                Yl = Y[..., :F].double()
                u = 2.0 ** -24
                tm = 2 * 7 * u * Yl.abs().mean(dim=(0, 1, 2)).max().item() + 1e-12
                tv = 2 * 7 * u * (Yl * Yl).mean(dim=(0, 1, 2)).max().item() + 2 * mean_r.abs().max().item() * tm + 1e-12
                assert (mean - mean_r).abs().max().item() <= tm, f"{tag}: BN mean"
                assert (var - var_r).abs().max().item() <= tv, f"{tag}: BN var"
            # (4b) BN statistics fused into the overlapped forward (interior and
            # boundary launches each contribute partial slots)
            y3 = torch.empty_like(y)
            xb.copy_(fill_owned_only(x, xd))
            torch.cuda.synchronize()
            dist.barrier()
            dc.dc_conv_fwd(plan, xb.data_ptr(), wb, y3, dc.DC_EXCHANGE | dc.DC_BN_STATS)
            m3, v3 = torch.zeros_like(mean), torch.zeros_like(var)
            dc.dc_bn_spatial_stats(plan, y3, m3, v3, dc.DC_BN_FROM_FWD)
            torch.cuda.synchronize()
            assert torch.equal(y3, ys), f"{tag}: y (fused BN) not bitwise equal to 1-GPU"
            # fused path: <= 2 x 16 in-register fp32 adds + depth-5 warp tree, DESIGN.md §7
            yl = y3[..., :F].double()
            u = 2.0 ** -24
            tm = 40 * u * yl.abs().mean(dim=(0, 1, 2)).max().item() + 1e-12
            tv = 40 * u * (yl * yl).mean(dim=(0, 1, 2)).max().item() + 2 * mean.abs().max().item() * tm + 1e-12
            assert (m3 - mean).abs().max().item() <= 4 * tm and (v3 - var).abs().max().item() <= 4 * tv, \
                f"{tag}: fused BN statistics differ"
            # (5) repeated BN calls cycle the P2P mailbox parities; results identical
            for _ in range(3):
                m2, v2 = torch.zeros_like(mean), torch.zeros_like(var)
                dc.dc_bn_spatial_stats(plan, y, m2, v2, False)
                torch.cuda.synchronize()
                assert torch.equal(m2, mean) and torch.equal(v2, var), f"{tag}: repeated BN differs"
            # (6) dW allreduce queued on the gradient stream, joined by dc_comm_sync
            dw2 = torch.empty_like(dw)
            dist.barrier()
            dc.dc_conv_bwd(plan, xb.data_ptr(), dyb.data_ptr(), wb, dx, dw2,
                           dc.DC_DEFAULT_FLAGS | dc.DC_ALLREDUCE_ASYNC)
            dc.dc_comm_sync(comm)
            torch.cuda.synchronize()
            e = rel_max(dw_to_fckk(dw2, C), dw_to_fckk(DW, C))
            assert e <= 1e-4, f"{tag}: async dW rel err {e}"
            assert torch.equal(dx, dxs), f"{tag}: dx (async allreduce) not bitwise equal to 1-GPU"
            # (7) the P2P protocol replayed from CUDA graphs (device-side epochs)
            s = torch.cuda.Stream()
            y2 = torch.empty_like(y)
            torch.cuda.synchronize()
            dist.barrier()
            with torch.cuda.stream(s):
                g_ex, g_fwd = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
                with torch.cuda.graph(g_ex, stream=s):
                    dc.dc_halo_exchange(plan, dc.DC_X, xb, 0)
                with torch.cuda.graph(g_fwd, stream=s):
                    dc.dc_conv_fwd(plan, xb.data_ptr(), wb, y2, dc.DC_EXCHANGE)
                for rep in range(3):
                    xb.copy_(fill_owned_only(x, xd))
                    torch.cuda.synchronize()
                    dist.barrier()
                    g_ex.replay()
                    torch.cuda.synchronize()
                    assert torch.equal(xb, full_x), f"{tag}: graph replay {rep}: x halo not bit-exact"
                    xb.copy_(fill_owned_only(x, xd))
                    y2.zero_()
                    torch.cuda.synchronize()
                    dist.barrier()
                    g_fwd.replay()
                    torch.cuda.synchronize()
                    assert torch.equal(y2, ys), f"{tag}: graph replay {rep}: y not bitwise equal"
            dist.barrier()
            dc.dc_plan_destroy(plan)
            dc.dc_plan_destroy(ref)
        dc.dc_comm_destroy(comm)
        dist.destroy_process_group()
    except Exception:
        errq.put(f"rank {rank}: {traceback.format_exc()}")
        raise


@pytest.mark.parametrize("world,env", [(2, None), (4, None)])
def test_multigpu_parity(world, env):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, errq, env)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    for p in procs:
        if p.is_alive():
            p.kill()
            errs.append("timeout")
    assert not errs and all(p.exitcode == 0 for p in procs), "\n".join(errs)
