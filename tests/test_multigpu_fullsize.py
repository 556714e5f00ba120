"""Multi-GPU parity at the bench's FULL sizes (mesh2k_n8 layers, N = 8), one
process per GPU over the P2P halo exchange, the NCCL dW allreduce and the
NVLink BN allreduce, with the flags bench.py times. Run under
`gpurun --gpus 2|4`.

Per rank, on sampled outputs the fp64 oracle computes one by one (the
row-window identities of tests/test_gpu_fullsize.py, pinned on CPU by
tests/test_fullsize_windows.py):
  * the first and last OWNED rows of y and dx (the rows that read the halo
    received from the neighbour: Eq. 1 / Eq. 3 across the partition seam,
    PAPER.md:137-141), owned columns, first and last sample;
  * dW (allreduced over all ranks) entries against Eq. 2;
  * the spatially aggregated BN statistics against fp64 sums
    of the stored y of all ranks.
"""
import os
import socket
import traceback

import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

# (name, N, C, H, W, F, K, S, P), grid
CASES = {
    2: [(("conv1_2", 8, 64, 1024, 1024, 64, 3, 1, 1), (1, 2, 1)),
        (("conv2_1", 8, 64, 1024, 1024, 128, 3, 2, 1), (1, 2, 1)),
        (("conv4_2", 8, 512, 128, 128, 512, 3, 1, 1), (1, 1, 2))],
    4: [(("conv1_2", 8, 64, 1024, 1024, 64, 3, 1, 1), (1, 4, 1)),
        (("conv3_2", 8, 256, 256, 256, 256, 3, 1, 1), (1, 2, 2)),
        (("conv1_1", 8, 18, 2048, 2048, 64, 3, 2, 1), (1, 4, 1))],
}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rel_l2(g, o):
    return float(np.linalg.norm((g - o).ravel()) / max(np.linalg.norm(o.ravel()), 1e-300))


def _worker(rank, world, port, errq):
    try:
        import sys
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, root)
        import torch.distributed as dist
        import datagen
        import oracle
        import paper_1903_06681_b200 as dc
        from tests.test_gpu_fullsize import _bwd_window, _fwd_window
        torch.cuda.set_device(rank)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        uid = [dc.dc_comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = dc.dc_comm_create(rank, world, uid[0], rank)
        for (name, N, C, H, W, F, K, S, P), grid in CASES[world]:
            tag = f"rank {rank} {name} grid {grid}"
            Ho, Wo = oracle.out_extent(H, K, S, P), oracle.out_extent(W, K, S, P)
            plan = dc.dc_plan_create(N, C, H, W, F, K, S, P, grid, dc.DC_BF16, comm)
            xd, yd = dc.dc_plan_query(plan, dc.DC_X), dc.dc_plan_query(plan, dc.DC_Y)
            dyd, dxd = dc.dc_plan_query(plan, dc.DC_DY), dc.dc_plan_query(plan, dc.DC_DX)
            xb = dc.wrap_device_buffer(dc.dc_buffer_alloc(plan, dc.DC_X), (xd["n"], xd["hb"], xd["wb"], xd["c_pad"]))
            dyb = dc.wrap_device_buffer(dc.dc_buffer_alloc(plan, dc.DC_DY),
                                        (dyd["n"], dyd["hb"], dyd["wb"], dyd["c_pad"]))

            def owned(desc, tid, shape):  # as bench.py: the generator on the GPU, owned block only
                return datagen.gen_block_nhwc_torch(
                    shape, datagen.SEED, tid, n=(desc["n0"], desc["n0"] + desc["n"]),
                    h=(desc["h0"], desc["h0"] + desc["h"]), w=(desc["w0"], desc["w0"] + desc["w"]),
                    c_pad=desc["c_pad"], dtype=torch.bfloat16, device="cuda")

            xb.zero_()
            dyb.zero_()
            xb[:, xd["halo_n"]:xd["halo_n"] + xd["h"], xd["halo_w"]:xd["halo_w"] + xd["w"]] = \
                owned(xd, datagen.TID_X, (N, C, H, W))
            dyb[:, dyd["halo_n"]:dyd["halo_n"] + dyd["h"], dyd["halo_w"]:dyd["halo_w"] + dyd["w"]] = \
                owned(dyd, datagen.TID_DY, (N, F, Ho, Wo))
            w = datagen.gen_w(F, C, K)
            wnp = np.zeros((F, K, K, xd["c_pad"]))
            wnp[..., :C] = w.transpose(0, 2, 3, 1)
            wb = torch.tensor(wnp, dtype=torch.bfloat16, device="cuda").contiguous()
            y = torch.empty((yd["n"], yd["h"], yd["w"], yd["c_pad"]), dtype=torch.bfloat16, device="cuda")
            dx = torch.empty((dxd["n"], dxd["h"], dxd["w"], dxd["c_pad"]), dtype=torch.bfloat16, device="cuda")
            dw = torch.empty((F, K, K, C), dtype=torch.float32, device="cuda")
            mean = torch.zeros(F, dtype=torch.float64, device="cuda")
            var = torch.zeros(F, dtype=torch.float64, device="cuda")
            torch.cuda.synchronize()
            dist.barrier()
            dc.dc_conv_fwd(plan, xb.data_ptr(), wb, y, dc.DC_EXCHANGE | dc.DC_BN_STATS)
            dc.dc_bn_spatial_stats(plan, y, mean, var, dc.DC_BN_FROM_FWD)
            dc.dc_conv_bwd(plan, xb.data_ptr(), dyb.data_ptr(), wb, dx, dw, dc.DC_DEFAULT_FLAGS)
            torch.cuda.synchronize()

            # spatial BN statistics vs fp64 sums of every rank's stored y
            y64 = y[..., :F].double()
            sums = torch.stack([y64.sum(dim=(0, 1, 2)), (y64 * y64).sum(dim=(0, 1, 2)),
                                y64.abs().sum(dim=(0, 1, 2))]).cpu()
            cnt = torch.tensor([float(y64.shape[0] * y64.shape[1] * y64.shape[2])], dtype=torch.float64)
            del y64
            dist.all_reduce(sums)
            dist.all_reduce(cnt)
            m_ref = (sums[0] / cnt).numpy()
            ex2 = (sums[1] / cnt).numpy()
            v_ref = ex2 - m_ref * m_ref
            u = 2.0 ** -24
            tm = 2 * 40 * u * (sums[2] / cnt).numpy() + 1e-12  # two groupings of the fused depth-40 sums (§7)
            tv = 2 * 40 * u * ex2 + 2 * np.abs(m_ref) * tm + 1e-9
            assert (np.abs(mean.cpu().numpy() - m_ref) <= tm).all(), f"{tag}: BN mean"
            assert (np.abs(var.cpu().numpy() - v_ref) <= tv).all(), f"{tag}: BN var"

            # first / last owned rows of y and dx (the halo-dependent seam rows)
            for n in (0, N - 1):
                if not (yd["n0"] <= n < yd["n0"] + yd["n"]):
                    continue
                nl = n - yd["n0"]
                for il in sorted({0, yd["h"] - 1}):
                    i = yd["h0"] + il
                    r0, L, ip = _fwd_window(i, H, K, S, P)
                    xw = datagen.gen_x(N, C, H, W, n=(n, n + 1), h=(r0, r0 + L))
                    ref = oracle.conv_fwd(xw, w, S, P, rows=(ip, ip + 1))[0, :, ip, yd["w0"]:yd["w0"] + yd["w"]]
                    got = y[nl, il, :, :F].double().cpu().numpy().T
                    e = _rel_l2(got, ref)
                    assert e <= 4e-3, f"{tag}: y[{n}, :, {i}, owned cols] rel L2 {e:.2e}"
                for ul in sorted({0, dxd["h"] - 1}):
                    uu = dxd["h0"] + ul
                    i0, i1, Hl, up = _bwd_window(uu, Ho, H, K, S, P)
                    dyw = datagen.gen_dy(N, F, Ho, Wo, n=(n, n + 1), h=(i0, i1))
                    ref = oracle.conv_bwd_data(dyw, w, Hl, W, S, P, rows=(up, up + 1))[0, :, up,
                                                                                      dxd["w0"]:dxd["w0"] + dxd["w"]]
                    got = dx[nl, ul, :, :C].double().cpu().numpy().T
                    e = _rel_l2(got, ref)
                    assert e <= 4e-3, f"{tag}: dx[{n}, :, {uu}, owned cols] rel L2 {e:.2e}"

            # allreduced dW (the same on every rank): two entries on rank 0
            if rank == 0:
                dwh = dw[..., :C].double().cpu().numpy()
                got, ref = [], []
                for f, c, a, b in ((0, 0, 0, 0), (F - 1, C - 1, K - 1, K - 1)):
                    xc = datagen.gen_x(N, C, H, W, c=(c, c + 1))
                    dyf = datagen.gen_dy(N, F, Ho, Wo, c=(f, f + 1))
                    ref.append(oracle.conv_bwd_filter_entry(xc, dyf, K, S, P, 0, 0, a, b))
                    got.append(dwh[f, a, b, c])
                got, ref = np.array(got), np.array(ref)
                e = np.abs(got - ref).max() / np.abs(ref).max()
                assert e <= 1e-4, f"{tag}: dW sampled {got} vs {ref}: {e:.2e}"
            torch.cuda.synchronize()
            dist.barrier()
            del xb, dyb
            dc.dc_plan_destroy(plan)
        dc.dc_comm_destroy(comm)
        dist.destroy_process_group()
    except Exception:
        errq.put(f"rank {rank}: {traceback.format_exc()}")
        raise


@pytest.mark.parametrize("world", [2, 4])
def test_multigpu_fullsize_sampled(world):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=900)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    for p in procs:
        if p.is_alive():
            p.kill()
            errs.append("timeout")
    assert not errs and all(p.exitcode == 0 for p in procs), "\n".join(errs)
