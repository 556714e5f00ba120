"""Channel / filter parallelism:
dc_cplan_* / dc_cconv_*.

CPU (virtual plans): every rank's shards are the blocks the paper's
distribution assigns -- x / dx / dW on the input-channel block i_C, y / dy on
the filter block i_C, samples on block i_N -- and the blocks of
a p_N x p_C grid tile every tensor exactly once (oracle.partition.blocked).

GPU (loopback group, virtual ranks on one device): the forward's
reduce-scatter over F and the backward-data's reduce-scatter over C (fused
into the conv GEMM epilogue) and the backward-filter's gather of
dy give every rank's y / dx / dW block within the element-wise error bound
 of the oracle's fp64 result; repeated calls and CUDA-graph
replay keep the device epochs in step."""
import numpy as np
import pytest
import torch

import datagen
import oracle
from oracle import partition as part
from tests.gpu_util import assert_elementwise, elementwise_bound


@pytest.fixture(scope="module")
def dc():
    from paper_1903_06681_b200 import build
    build.build()
    import paper_1903_06681_b200 as dc
    return dc


GEOM = [((4, 64, 16, 16, 128, 3, 1, 1), 2, 2), ((2, 128, 12, 12, 64, 3, 2, 1), 1, 4),
        ((3, 256, 8, 8, 512, 1, 1, 0), 3, 8)]


@pytest.mark.parametrize("shape,pn,pc", GEOM)
def test_cplan_shards_are_the_papers_blocks(dc, shape, pn, pc):
    N, C, H, W, F, K, S, P = shape
    Ho, Wo = oracle.out_extent(H, K, S, P), oracle.out_extent(W, K, S, P)
    seen = {t: np.zeros(n, dtype=int) for t, n in (("x", N * C), ("y", N * F))}
    for rank in range(pn * pc):
        i_n, i_c = divmod(rank, pc)
        plan = dc.dc_cplan_create_virtual(*shape, pn, pc, rank)
        try:
            n0, n1 = part.blocked(N, pn, i_n)
            c0, c1 = part.blocked(C, pc, i_c)
            f0, f1 = part.blocked(F, pc, i_c)
            for t, (h, w, lo, hi) in ((dc.DC_X, (H, W, c0, c1)), (dc.DC_DX, (H, W, c0, c1)),
                                      (dc.DC_Y, (Ho, Wo, f0, f1)), (dc.DC_DY, (Ho, Wo, f0, f1))):
                d = dc.dc_cplan_query(plan, t)
                assert (d["n0"], d["n"], d["h0"], d["h"], d["w0"], d["w"]) == (n0, n1 - n0, 0, h, 0, w)
                assert (d["c0"], d["c"], d["c_pad"]) == (lo, hi - lo, hi - lo)
                assert d["halo_n"] == d["halo_s"] == d["halo_w"] == d["halo_e"] == 0
                assert d["bytes"] == (n1 - n0) * h * w * (hi - lo) * 2
            for n in range(n0, n1):
                seen["x"][n * C + c0:n * C + c1] += 1
                seen["y"][n * F + f0:n * F + f1] += 1
            d = dc.dc_cplan_query(plan, dc.DC_DW)
            assert (d["n"], d["h"], d["w"], d["c"], d["c0"]) == (F, K, K, c1 - c0, c0)
            d = dc.dc_cplan_query(plan, dc.DC_W)
            assert (d["n"], d["c"], d["c0"], d["bytes"]) == (F, C, 0, F * K * K * C * 2)
        finally:
            dc.dc_cplan_destroy(plan)
    assert (seen["x"] == 1).all() and (seen["y"] == 1).all()


def test_cplan_errors(dc):
    with pytest.raises(dc.DCError):   # C not a multiple of 16 p_C
        dc.dc_cplan_create_virtual(2, 48, 8, 8, 64, 3, 1, 1, 1, 2, 0)
    with pytest.raises(dc.DCError):   # more sample blocks than samples
        dc.dc_cplan_create_virtual(2, 64, 8, 8, 64, 3, 1, 1, 4, 2, 0)
    with pytest.raises(dc.DCError):   # p_C > 8
        dc.dc_cplan_create_virtual(2, 256, 8, 8, 256, 3, 1, 1, 1, 16, 0)
    with pytest.raises(dc.DCError):   # rank outside the grid
        dc.dc_cplan_create_virtual(2, 64, 8, 8, 64, 3, 1, 1, 1, 2, 2)
    with pytest.raises(dc.DCError):   # fp32 plans
        dc.dc_cplan_create(2, 64, 8, 8, 64, 3, 1, 1, 1, 1, dc.DC_FP32_3XTF32, None)
    p = dc.dc_cplan_create_virtual(2, 64, 8, 8, 64, 3, 1, 1, 1, 2, 0)
    try:
        with pytest.raises(dc.DCError):   # virtual plans carry no data
            dc.dc_cconv_fwd(p, 1, 2, 3, 0, 0)
    finally:
        dc.dc_cplan_destroy(p)


# ---------------------------------------------------------------------------
# GPU: loopback group
# ---------------------------------------------------------------------------
CASES = [
    ((2, 64, 16, 16, 64, 3, 1, 1), 1, 2),
    ((2, 128, 12, 12, 64, 3, 1, 1), 1, 4),
    ((4, 64, 16, 16, 128, 3, 1, 1), 2, 2),      # hybrid sample x channel
    ((2, 64, 18, 18, 64, 3, 2, 1), 1, 2),       # stride 2: backward-data phase GEMMs
    ((2, 256, 8, 8, 256, 1, 1, 0), 1, 2),       # 1x1
    ((1, 512, 16, 16, 512, 3, 1, 1), 1, 8),     # deep layer, 8 ranks (split-K partials)
]


def _nhwc(t, c0, c1, n0, n1):
    """Global NCHW float64 -> bf16 NHWC block [n0:n1, ..., c0:c1] on the GPU."""
    return torch.tensor(t[n0:n1, c0:c1].transpose(0, 2, 3, 1), dtype=torch.bfloat16, device="cuda").contiguous()


def _to_nchw(t):
    return t.float().cpu().numpy().astype(np.float64).transpose(0, 3, 1, 2)


@pytest.mark.gpu
@pytest.mark.parametrize("shape,pn,pc", CASES)
def test_loopback_channel_parallel_parity(dc, shape, pn, pc):
    N, C, H, W, F, K, S, P = shape
    Ho, Wo = oracle.out_extent(H, K, S, P), oracle.out_extent(W, K, S, P)
    x, w, dy = datagen.gen_x(N, C, H, W), datagen.gen_w(F, C, K), datagen.gen_dy(N, F, Ho, Wo)
    y_ref, dx_ref = oracle.conv_fwd(x, w, S, P), oracle.conv_bwd_data(dy, w, H, W, S, P)
    ax, aw, ady = np.abs(x), np.abs(w), np.abs(dy)
    y_abs, dx_abs = oracle.conv_fwd(ax, aw, S, P), oracle.conv_bwd_data(ady, aw, H, W, S, P)
    wb = torch.tensor(w.transpose(0, 2, 3, 1), dtype=torch.bfloat16, device="cuda").contiguous()
    world = pn * pc
    comms = dc.dc_comm_create_local(world, torch.cuda.current_device())
    R = []
    try:
        for rank, comm in enumerate(comms):
            plan = dc.dc_cplan_create(*shape, pn, pc, dc.DC_BF16, comm)
            q = {t: dc.dc_cplan_query(plan, t) for t in (dc.DC_X, dc.DC_Y, dc.DC_DX, dc.DC_DY, dc.DC_DW)}
            n0, nn = q[dc.DC_X]["n0"], q[dc.DC_X]["n"]
            cx, cy = q[dc.DC_X], q[dc.DC_Y]
            R.append(dict(
                plan=plan, q=q, n0=n0, n1=n0 + nn, stream=torch.cuda.ExternalStream(dc.dc_comm_stream(comm)),
                x=_nhwc(x, cx["c0"], cx["c0"] + cx["c"], n0, n0 + nn),
                dy=_nhwc(dy, cy["c0"], cy["c0"] + cy["c"], n0, n0 + nn),
                y=torch.full((nn, Ho, Wo, cy["c"]), float("nan"), dtype=torch.bfloat16, device="cuda"),
                dx=torch.full((nn, H, W, cx["c"]), float("nan"), dtype=torch.bfloat16, device="cuda"),
                dw=torch.full((F, K, K, cx["c"]), float("nan"), dtype=torch.float32, device="cuda")))
        torch.cuda.synchronize()

        def step(d):
            dc.dc_cconv_fwd(d["plan"], d["x"], wb, d["y"], 0, d["stream"])
            dc.dc_cconv_bwd_data(d["plan"], d["dy"], wb, d["dx"], 0, d["stream"])
            dc.dc_cconv_bwd_filter(d["plan"], d["x"], d["dy"], d["dw"], 0, d["stream"])

        def run_all(fn):
            for d in R:
                with torch.cuda.stream(d["stream"]):
                    fn(d)
            torch.cuda.synchronize()

        def check(tag):
            for rank, d in enumerate(R):
                cx, cy = d["q"][dc.DC_X], d["q"][dc.DC_Y]
                n0, n1 = d["n0"], d["n1"]
                fs, cs = slice(cy["c0"], cy["c0"] + cy["c"]), slice(cx["c0"], cx["c0"] + cx["c"])
                assert_elementwise(f"{tag} rank {rank} y", _to_nchw(d["y"]), y_ref[n0:n1, fs],
                                   elementwise_bound(y_ref[n0:n1, fs], y_abs[n0:n1, fs], C * K * K, 16, True,
                                                     extra_adds=32 + pc))
                assert_elementwise(f"{tag} rank {rank} dx", _to_nchw(d["dx"]), dx_ref[n0:n1, cs],
                                   elementwise_bound(dx_ref[n0:n1, cs], dx_abs[n0:n1, cs], F * K * K, 16, True,
                                                     extra_adds=32 + pc))
                # dW of the rank's samples (the p_N sample groups' sum is DC_ALLREDUCE, real ranks)
                dw_ref = oracle.conv_bwd_filter(x[n0:n1], dy[n0:n1], K, S, P)[:, cs]
                dw_abs = oracle.conv_bwd_filter(ax[n0:n1], ady[n0:n1], K, S, P)[:, cs]
                dw = d["dw"].double().cpu().numpy().transpose(0, 3, 1, 2)
                assert_elementwise(f"{tag} rank {rank} dw", dw, dw_ref,
                                   elementwise_bound(dw_ref, dw_abs, (n1 - n0) * Ho * Wo, 16, False, extra_adds=300))

        run_all(step)
        check("eager")
        run_all(step)     # second epoch
        check("epoch 2")
        graphs = []
        for d in R:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(d["stream"]):
                with torch.cuda.graph(g, stream=d["stream"]):
                    step(d)
            graphs.append(g)
        torch.cuda.synchronize()
        for d in R:
            d["y"].fill_(float("nan")), d["dx"].fill_(float("nan")), d["dw"].fill_(float("nan"))
        torch.cuda.synchronize()
        for d, g in zip(R, graphs):
            with torch.cuda.stream(d["stream"]):
                g.replay()
        torch.cuda.synchronize()
        check("replay")
    finally:
        for d in R:
            dc.dc_cplan_destroy(d["plan"])
        for c in comms:
            dc.dc_comm_destroy(c)


# ---------------------------------------------------------------------------
# GPU: real ranks (one process per GPU; CUDA-IPC peer memory, NCCL dW sum)
# ---------------------------------------------------------------------------
MG = {2: [((2, 64, 16, 16, 64, 3, 1, 1), 1, 2), ((4, 64, 12, 12, 64, 3, 1, 1), 2, 1)],
      4: [((4, 64, 16, 16, 128, 3, 1, 1), 2, 2), ((2, 128, 12, 12, 64, 3, 2, 1), 1, 4)]}


def _mg_worker(rank, world, port, errq):
    import os
    import sys
    import traceback
    try:
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, root)
        import torch.distributed as dist
        import paper_1903_06681_b200 as dc
        torch.cuda.set_device(rank)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        uid = [dc.dc_comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = dc.dc_comm_create(rank, world, uid[0], rank)
        for shape, pn, pc in MG[world]:
            N, C, H, W, F, K, S, P = shape
            Ho, Wo = oracle.out_extent(H, K, S, P), oracle.out_extent(W, K, S, P)
            x, w, dy = datagen.gen_x(N, C, H, W), datagen.gen_w(F, C, K), datagen.gen_dy(N, F, Ho, Wo)
            wb = torch.tensor(w.transpose(0, 2, 3, 1), dtype=torch.bfloat16, device="cuda").contiguous()
            plan = dc.dc_cplan_create(*shape, pn, pc, dc.DC_BF16, comm)
            cx, cy = dc.dc_cplan_query(plan, dc.DC_X), dc.dc_cplan_query(plan, dc.DC_Y)
            n0, n1 = cx["n0"], cx["n0"] + cx["n"]
            xs = _nhwc(x, cx["c0"], cx["c0"] + cx["c"], n0, n1)
            dys = _nhwc(dy, cy["c0"], cy["c0"] + cy["c"], n0, n1)
            y = torch.empty((n1 - n0, Ho, Wo, cy["c"]), dtype=torch.bfloat16, device="cuda")
            dx = torch.empty((n1 - n0, H, W, cx["c"]), dtype=torch.bfloat16, device="cuda")
            dw = torch.empty((F, K, K, cx["c"]), dtype=torch.float32, device="cuda")
            for _ in range(2):
                torch.cuda.synchronize()
                dist.barrier()
                dc.dc_cconv_fwd(plan, xs, wb, y)
                dc.dc_cconv_bwd_data(plan, dys, wb, dx)
                dc.dc_cconv_bwd_filter(plan, xs, dys, dw, dc.DC_ALLREDUCE)
                torch.cuda.synchronize()
            fs, cs = slice(cy["c0"], cy["c0"] + cy["c"]), slice(cx["c0"], cx["c0"] + cx["c"])
            tag = f"rank {rank} {shape} ({pn},{pc})"
            y_ref = oracle.conv_fwd(x, w, S, P)[n0:n1, fs]
            assert_elementwise(f"{tag} y", _to_nchw(y), y_ref, elementwise_bound(
                y_ref, oracle.conv_fwd(np.abs(x), np.abs(w), S, P)[n0:n1, fs], C * K * K, 16, True, 32 + pc))
            dx_ref = oracle.conv_bwd_data(dy, w, H, W, S, P)[n0:n1, cs]
            assert_elementwise(f"{tag} dx", _to_nchw(dx), dx_ref, elementwise_bound(
                dx_ref, oracle.conv_bwd_data(np.abs(dy), np.abs(w), H, W, S, P)[n0:n1, cs], F * K * K, 16, True,
                32 + pc))
            dw_ref = oracle.conv_bwd_filter(x, dy, K, S, P)[:, cs]       # all samples: summed over i_N
            assert_elementwise(f"{tag} dw", dw.double().cpu().numpy().transpose(0, 3, 1, 2), dw_ref,
                               elementwise_bound(dw_ref, oracle.conv_bwd_filter(np.abs(x), np.abs(dy), K, S, P)[:, cs],
                                                 N * Ho * Wo, 16, False, extra_adds=300 + pn))
            dist.barrier()
            dc.dc_cplan_destroy(plan)
        dc.dc_comm_destroy(comm)
        dist.destroy_process_group()
    except Exception:
        errq.put(f"rank {rank}: {traceback.format_exc()}")
        raise


@pytest.mark.gpu
@pytest.mark.multigpu
@pytest.mark.parametrize("world", [2, 4])
def test_multigpu_channel_parallel(world):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    procs = [ctx.Process(target=_mg_worker, args=(r, world, port, errq)) for r in range(world)]
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
