"""Redistribution between decompositions (Shuffle(D_i, D_j), PAPER.md:151-153;
SURVEY.md 8(f) NEXT-3): dc_redist_create / dc_redistribute.

CPU (virtual plans): the bytes every rank sends to every other rank equal the
oracle's element-by-element ownership count (oracle/perfmodel.shuffle_words)
times the bytes per word of the padded pixel, and every element of the tensor
is kept or sent exactly once (conservation, send/recv duality).

GPU (loopback group, 2-8 virtual ranks on one device): the one-kernel P2P
all-to-all leaves every destination interior bitwise equal to the global
tensor's block and the margins untouched; chained between two layers of
different grids (layer A's y -> layer B's x, forward with DC_EXCHANGE, and
layer B's dx -> layer A's dy) the result is bitwise the 1-GPU chain's; repeated
and graph-replayed calls advance the device epochs."""
import numpy as np
import pytest
import torch

import datagen
import oracle
from oracle import perfmodel as pm
from tests.gpu_util import fill_buffer, weights_gpu


@pytest.fixture(scope="module")
def dc():
    from paper_1903_06681_b200 import build
    build.build()
    import paper_1903_06681_b200 as dc
    return dc


def _virtual_set(dc, shape, grid):
    N, C, H, W, F, K, S, P = shape
    world = grid[0] * grid[1] * grid[2]
    return [dc.dc_plan_create_virtual(N, C, H, W, F, K, S, P, grid, r) for r in range(world)]


# (N, Ch, H, W), grid A, grid B: an x -> x redistribution between two 3x3/1
# layers of the same input shape, whose x ownership is the blocked one the
# oracle's owner() assigns
X_CASES = [
    ((4, 16, 24, 20), (4, 1, 1), (1, 4, 1)),   # sample -> spatial (PAPER.md:153 example)
    ((4, 16, 24, 20), (1, 2, 2), (2, 2, 1)),
    ((2, 32, 33, 30), (1, 1, 2), (1, 2, 1)),   # W split -> H split, ragged
    ((3, 8, 20, 20), (1, 3, 1), (1, 1, 3)),
    ((6, 16, 12, 10), (2, 3, 1), (3, 1, 2)),
    ((8, 16, 16, 16), (8, 1, 1), (2, 2, 2)),   # 8 ranks
    ((2, 16, 20, 20), (1, 2, 1), (1, 2, 1)),   # same grid: each rank keeps its block
]


@pytest.mark.parametrize("ext,ga,gb", X_CASES)
def test_redist_bytes_match_oracle_ownership(dc, ext, ga, gb):
    N, Ch, H, W = ext
    A = _virtual_set(dc, (N, 16, H, W, Ch, 3, 1, 1), ga)   # y of A: N x Ch x H x W (3x3/1 same)
    B = _virtual_set(dc, (N, Ch, H, W, 16, 3, 1, 1), gb)   # x of B
    world = len(A)
    try:
        words = pm.shuffle_words(N, Ch, H, W, ga, gb)
        cpad = dc.dc_plan_query(B[0], dc.DC_X)["c_pad"]
        per_word = cpad * 2 / Ch                       # bf16 bytes moved per logical word
        send = np.zeros((world, world), dtype=np.int64)
        recv = np.zeros((world, world), dtype=np.int64)
        for r in range(world):
            for src_t in (dc.DC_Y,):
                h = dc.dc_redist_create(A[r], src_t, B[r], dc.DC_X)
                send[r], recv[r] = dc.dc_redist_bytes(h, world)
                dc.dc_redist_destroy(h)
        for r in range(world):
            for q in range(world):
                if r != q:
                    assert send[r, q] == words.get((r, q), 0) * per_word, (r, q)
        assert np.array_equal(send, recv.T)                              # duality
        assert send.sum() == N * H * W * cpad * 2                       # every element once
        kept = np.diag(send).sum()
        assert kept == N * H * W * cpad * 2 - sum(words.values()) * per_word
    finally:
        for p in A + B:
            dc.dc_plan_destroy(p)


def test_redist_strided_source_conserves(dc):
    """y of a stride-2 layer (ownership derived from the owned inputs,
    PAPER.md:137) into the x of a 3x3/1 layer of another grid: conservation
    and duality, and every rank's received bytes cover its owned x block."""
    A = _virtual_set(dc, (2, 16, 34, 30, 32, 3, 2, 1), (1, 4, 1))   # y: 2 x 32 x 17 x 15
    B = _virtual_set(dc, (2, 32, 17, 15, 16, 3, 1, 1), (1, 2, 2))
    world = 4
    try:
        send = np.zeros((world, world), dtype=np.int64)
        recv = np.zeros((world, world), dtype=np.int64)
        for r in range(world):
            h = dc.dc_redist_create(A[r], dc.DC_Y, B[r], dc.DC_X)
            send[r], recv[r] = dc.dc_redist_bytes(h, world)
            dc.dc_redist_destroy(h)
        assert np.array_equal(send, recv.T)
        assert send.sum() == 2 * 17 * 15 * 32 * 2
        for r in range(world):
            d = dc.dc_plan_query(B[r], dc.DC_X)
            assert recv[r].sum() == d["n"] * d["h"] * d["w"] * d["c_pad"] * 2
    finally:
        for p in A + B:
            dc.dc_plan_destroy(p)


def test_redist_errors(dc):
    a = dc.dc_plan_create_virtual(2, 16, 16, 16, 32, 3, 1, 1, (1, 2, 1), 0)
    b = dc.dc_plan_create_virtual(2, 32, 16, 16, 16, 3, 1, 1, (1, 1, 2), 0)
    c = dc.dc_plan_create_virtual(2, 16, 16, 16, 16, 3, 1, 1, (1, 1, 2), 0)
    f32a = dc.dc_plan_create_virtual(2, 16, 16, 16, 32, 3, 1, 1, (1, 2, 1), 0, dc.DC_FP32_3XTF32)
    f32b = dc.dc_plan_create_virtual(2, 32, 16, 16, 16, 3, 1, 1, (1, 1, 2), 0, dc.DC_FP32_3XTF32)
    try:
        with pytest.raises(dc.DCError):          # channel counts differ (y of a: 32, x of c: 16)
            dc.dc_redist_create(a, dc.DC_Y, c, dc.DC_X)
        with pytest.raises(dc.DCError):          # the destination is an activation / gradient
            dc.dc_redist_create(a, dc.DC_Y, b, dc.DC_W)
        with pytest.raises(dc.DCError):          # fp32: dense y -> split [hi | lo] x
            dc.dc_redist_create(f32a, dc.DC_Y, f32b, dc.DC_X)
        with pytest.raises(dc.DCError):          # mixed dtypes
            dc.dc_redist_create(a, dc.DC_Y, f32b, dc.DC_X)
        h = dc.dc_redist_create(a, dc.DC_Y, b, dc.DC_X)
        with pytest.raises(dc.DCError):          # virtual plans carry no data
            dc.dc_redistribute(h, 1, 2, 0, 0)
        dc.dc_redist_destroy(h)
    finally:
        for p in (a, b, c, f32a, f32b):
            dc.dc_plan_destroy(p)


# ---------------------------------------------------------------------------
# GPU: loopback group
# ---------------------------------------------------------------------------
# layer A (N, C0, HA, WA, F=Ch, K, S, P) on grid A, layer B (N, Ch, H, W, F2, 3, 1, 1)
# on grid B, H x W = A's output
CHAIN = [
    ((4, 16, 24, 20, 16, 3, 1, 1), (4, 1, 1), (1, 4, 1), 32),
    ((2, 16, 33, 30, 32, 3, 1, 1), (1, 1, 2), (1, 2, 1), 16),
    ((4, 16, 24, 20, 16, 3, 1, 1), (1, 2, 2), (2, 2, 1), 16),
    ((2, 16, 34, 30, 32, 3, 2, 1), (1, 4, 1), (1, 2, 2), 64),   # strided producer
    ((8, 16, 16, 16, 16, 3, 1, 1), (8, 1, 1), (2, 2, 2), 16),   # 8 ranks
    ((2, 64, 16, 16, 64, 1, 1, 0), (2, 1, 1), (1, 1, 2), 64),
]


def _layer_b(shape_a, F2):
    N, C0, H, W, F, K, S, P = shape_a
    return (N, F, oracle.out_extent(H, K, S, P), oracle.out_extent(W, K, S, P), F2, 3, 1, 1)


class Group:
    def __init__(self, dc, shape_a, ga, shape_b, gb):
        self.dc = dc
        self.world = ga[0] * ga[1] * ga[2]
        self.comms = dc.dc_comm_create_local(self.world, torch.cuda.current_device())
        self.r = []
        for rank, comm in enumerate(self.comms):
            pa = dc.dc_plan_create(*shape_a, ga, dc.DC_BF16, comm)
            pb = dc.dc_plan_create(*shape_b, gb, dc.DC_BF16, comm)
            d = dict(pa=pa, pb=pb, stream=torch.cuda.ExternalStream(dc.dc_comm_stream(comm)))
            for key, plan in (("a", pa), ("b", pb)):
                for t, name in ((dc.DC_X, "x"), (dc.DC_Y, "y"), (dc.DC_DY, "dy"), (dc.DC_DX, "dx")):
                    d[f"q{key}{name}"] = dc.dc_plan_query(plan, t)
            for key, plan in (("a", pa), ("b", pb)):
                for t, name in ((dc.DC_X, "x"), (dc.DC_DY, "dy")):
                    q = d[f"q{key}{name}"]
                    d[f"{key}{name}b"] = dc.wrap_device_buffer(dc.dc_buffer_alloc(plan, t),
                                                               (q["n"], q["hb"], q["wb"], q["c_pad"]))
            self.r.append(d)
        # created after every rank's buffers exist (they are resolved at the first call)
        for d in self.r:
            d["fwd"] = dc.dc_redist_create(d["pa"], dc.DC_Y, d["pb"], dc.DC_X)
            d["bwd"] = dc.dc_redist_create(d["pb"], dc.DC_DX, d["pa"], dc.DC_DY)

    def each(self, fn):
        for d in self.r:
            with torch.cuda.stream(d["stream"]):
                fn(d)
        torch.cuda.synchronize()

    def close(self):
        for d in self.r:
            self.dc.dc_redist_destroy(d["fwd"])
            self.dc.dc_redist_destroy(d["bwd"])
            self.dc.dc_plan_destroy(d["pa"])
            self.dc.dc_plan_destroy(d["pb"])
        for c in self.comms:
            self.dc.dc_comm_destroy(c)


def _dense(q, glob_nhwc):
    """The owned block of a global NHWC (padded) tensor as a dense shard."""
    return glob_nhwc[q["n0"]:q["n0"] + q["n"], q["h0"]:q["h0"] + q["h"], q["w0"]:q["w0"] + q["w"]].contiguous()


@pytest.mark.gpu
@pytest.mark.parametrize("shape_a,ga,gb,F2", CHAIN)
def test_loopback_redistribute_bitexact(dc, shape_a, ga, gb, F2):
    """Y (dense, grid A) -> margined X (grid B) and DX (grid B) -> margined DY
    (grid A): interiors bitwise equal to the global tensor, margins untouched
    (sentinel), three epochs in a row."""
    shape_b = _layer_b(shape_a, F2)
    G = Group(dc, shape_a, ga, shape_b, gb)
    try:
        g = torch.Generator().manual_seed(1903)
        q0 = G.r[0]
        for epoch in range(3):
            Y = torch.randn((shape_b[0], shape_b[2], shape_b[3], q0["qay"]["c_pad"]), generator=g)
            Y = Y.to(torch.bfloat16).cuda()
            DX = torch.randn((shape_b[0], shape_b[2], shape_b[3], q0["qbdx"]["c_pad"]), generator=g)
            DX = DX.to(torch.bfloat16).cuda()
            for d in G.r:
                d["y"], d["dx"] = _dense(d["qay"], Y), _dense(d["qbdx"], DX)
                d["bxb"].fill_(7.0)
                d["adyb"].fill_(-3.0)
            torch.cuda.synchronize()
            G.each(lambda d: dc.dc_redistribute(d["fwd"], d["y"], d["bxb"], 0, d["stream"]))
            G.each(lambda d: dc.dc_redistribute(d["bwd"], d["dx"], d["adyb"], 0, d["stream"]))
            for rank, d in enumerate(G.r):
                for buf, q, glob, fill in ((d["bxb"], d["qbx"], Y, 7.0), (d["adyb"], d["qady"], DX, -3.0)):
                    hn, hw = q["halo_n"], q["halo_w"]
                    inner = buf[:, hn:hn + q["h"], hw:hw + q["w"]]
                    assert torch.equal(inner, _dense(q, glob)), f"epoch {epoch} rank {rank}: interior"
                    mask = torch.ones(buf.shape[:3], dtype=torch.bool, device=buf.device)
                    mask[:, hn:hn + q["h"], hw:hw + q["w"]] = False
                    assert bool((buf[mask] == fill).all()), f"epoch {epoch} rank {rank}: margin written"
    finally:
        G.close()


@pytest.mark.gpu
@pytest.mark.parametrize("shape_a,ga,gb,F2", [CHAIN[0], CHAIN[3], CHAIN[4]])
def test_loopback_redistributed_chain_bitwise(dc, shape_a, ga, gb, F2):
    """Two layers on different grids joined by redistributions: layer A
    forward (DC_EXCHANGE) -> y -> layer B's x -> layer B forward (DC_EXCHANGE,
    halo from B's neighbours) equals the 1-GPU chain bitwise; backward, B's
    dx -> A's dy -> A's backward-data equals the 1-GPU dx bitwise. Then the
    same step replayed from CUDA graphs."""
    shape_b = _layer_b(shape_a, F2)
    N, C0, H, W, F, K, S, P = shape_a
    x = datagen.gen_x(N, C0, H, W)
    wa = datagen.gen_w(F, C0, K)
    wbm = datagen.gen_w(F2, F, 3)
    dy2 = datagen.gen_dy(N, F2, shape_b[2], shape_b[3])
    # 1-GPU chain
    ref_a = dc.dc_plan_create_virtual(*shape_a, (1, 1, 1), 0)
    ref_b = dc.dc_plan_create_virtual(*shape_b, (1, 1, 1), 0)
    try:
        qa = {t: dc.dc_plan_query(ref_a, t) for t in (dc.DC_X, dc.DC_Y, dc.DC_DY, dc.DC_DX)}
        qb = {t: dc.dc_plan_query(ref_b, t) for t in (dc.DC_X, dc.DC_Y, dc.DC_DY, dc.DC_DX)}
        wa_g, wb_g = weights_gpu(wa, qa[dc.DC_X]["c_pad"]), weights_gpu(wbm, qb[dc.DC_X]["c_pad"])
        Y1 = torch.empty((N, qa[dc.DC_Y]["h"], qa[dc.DC_Y]["w"], qa[dc.DC_Y]["c_pad"]), dtype=torch.bfloat16,
                         device="cuda")
        dc.dc_conv_fwd(ref_a, fill_buffer(x, qa[dc.DC_X]), wa_g, Y1, 0)
        torch.cuda.synchronize()
        y1 = Y1[..., :F].double().cpu().numpy().transpose(0, 3, 1, 2)
        Y2 = torch.empty((N, qb[dc.DC_Y]["h"], qb[dc.DC_Y]["w"], qb[dc.DC_Y]["c_pad"]), dtype=torch.bfloat16,
                         device="cuda")
        dc.dc_conv_fwd(ref_b, fill_buffer(y1, qb[dc.DC_X]), wb_g, Y2, 0)
        DX2 = torch.empty((N, qb[dc.DC_DX]["h"], qb[dc.DC_DX]["w"], qb[dc.DC_DX]["c_pad"]), dtype=torch.bfloat16,
                          device="cuda")
        dc.dc_conv_bwd_data(ref_b, fill_buffer(dy2, qb[dc.DC_DY]), wb_g, DX2, 0)
        torch.cuda.synchronize()
        dx2 = DX2[..., :F].double().cpu().numpy().transpose(0, 3, 1, 2)
        DX1 = torch.empty((N, qa[dc.DC_DX]["h"], qa[dc.DC_DX]["w"], qa[dc.DC_DX]["c_pad"]), dtype=torch.bfloat16,
                          device="cuda")
        dc.dc_conv_bwd_data(ref_a, fill_buffer(dx2, qa[dc.DC_DY]), wa_g, DX1, 0)
        torch.cuda.synchronize()
    finally:
        dc.dc_plan_destroy(ref_a)
        dc.dc_plan_destroy(ref_b)

    G = Group(dc, shape_a, ga, shape_b, gb)
    try:
        for d in G.r:
            d["axb"].copy_(fill_buffer(x, d["qax"]))          # (margins re-filled by the exchange)
            d["bdyb"].copy_(fill_buffer(dy2, d["qbdy"]))
            d["y1"] = torch.empty((d["qay"]["n"], d["qay"]["h"], d["qay"]["w"], d["qay"]["c_pad"]),
                                  dtype=torch.bfloat16, device="cuda")
            d["y2"] = torch.empty((d["qby"]["n"], d["qby"]["h"], d["qby"]["w"], d["qby"]["c_pad"]),
                                  dtype=torch.bfloat16, device="cuda")
            d["dx2"] = torch.empty((d["qbdx"]["n"], d["qbdx"]["h"], d["qbdx"]["w"], d["qbdx"]["c_pad"]),
                                   dtype=torch.bfloat16, device="cuda")
            d["dx1"] = torch.empty((d["qadx"]["n"], d["qadx"]["h"], d["qadx"]["w"], d["qadx"]["c_pad"]),
                                   dtype=torch.bfloat16, device="cuda")
        torch.cuda.synchronize()

        def step(d):
            dc.dc_conv_fwd(d["pa"], d["axb"].data_ptr(), wa_g, d["y1"], dc.DC_EXCHANGE, d["stream"])
            dc.dc_redistribute(d["fwd"], d["y1"], d["bxb"], 0, d["stream"])
            dc.dc_conv_fwd(d["pb"], d["bxb"].data_ptr(), wb_g, d["y2"], dc.DC_EXCHANGE, d["stream"])
            dc.dc_conv_bwd_data(d["pb"], d["bdyb"].data_ptr(), wb_g, d["dx2"], dc.DC_EXCHANGE, d["stream"])
            dc.dc_redistribute(d["bwd"], d["dx2"], d["adyb"], 0, d["stream"])
            dc.dc_conv_bwd_data(d["pa"], d["adyb"].data_ptr(), wa_g, d["dx1"], dc.DC_EXCHANGE, d["stream"])

        def check(tag):
            for rank, d in enumerate(G.r):
                for got, q, ref, name in ((d["y2"], d["qby"], Y2, "y2"), (d["dx1"], d["qadx"], DX1, "dx1")):
                    assert torch.equal(got, _dense(q, ref)), f"{tag} rank {rank}: {name} not bitwise 1-GPU"

        G.each(step)
        check("eager")
        graphs = []
        for d in G.r:
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.stream(d["stream"]):
                with torch.cuda.graph(gr, stream=d["stream"]):
                    step(d)
            graphs.append(gr)
        torch.cuda.synchronize()
        for rep in range(2):
            for d in G.r:
                d["y2"].zero_(), d["dx1"].zero_()
            torch.cuda.synchronize()
            for d, gr in zip(G.r, graphs):
                with torch.cuda.stream(d["stream"]):
                    gr.replay()
            torch.cuda.synchronize()
            check(f"replay {rep}")
    finally:
        G.close()


# ---------------------------------------------------------------------------
# GPU: real ranks (one process per GPU; CUDA-IPC peer memory and NCCL)
# ---------------------------------------------------------------------------
MG_CASES = {
    2: [((4, 16, 24, 20, 16, 3, 1, 1), (2, 1, 1), (1, 2, 1), 32),
        ((2, 16, 34, 30, 32, 3, 2, 1), (1, 1, 2), (1, 2, 1), 64)],
    4: [((4, 16, 24, 20, 16, 3, 1, 1), (4, 1, 1), (1, 2, 2), 32),
        ((2, 16, 33, 30, 32, 3, 1, 1), (1, 4, 1), (2, 1, 2), 16)],
}


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
        for shape_a, ga, gb, F2 in MG_CASES[world]:
            shape_b = _layer_b(shape_a, F2)
            pa = dc.dc_plan_create(*shape_a, ga, dc.DC_BF16, comm)
            pb = dc.dc_plan_create(*shape_b, gb, dc.DC_BF16, comm)
            qay, qbx = dc.dc_plan_query(pa, dc.DC_Y), dc.dc_plan_query(pb, dc.DC_X)
            bxb = dc.wrap_device_buffer(dc.dc_buffer_alloc(pb, dc.DC_X), (qbx["n"], qbx["hb"], qbx["wb"], qbx["c_pad"]))
            r = dc.dc_redist_create(pa, dc.DC_Y, pb, dc.DC_X)
            g = torch.Generator().manual_seed(7)
            for transport in (0, dc.DC_HALO_NCCL, 0):
                Y = torch.randn((shape_b[0], shape_b[2], shape_b[3], qay["c_pad"]), generator=g)
                Y = Y.to(torch.bfloat16).cuda()
                y = _dense(qay, Y)
                bxb.fill_(5.0)
                torch.cuda.synchronize()
                dist.barrier()
                dc.dc_redistribute(r, y, bxb, transport)
                torch.cuda.synchronize()
                hn, hw = qbx["halo_n"], qbx["halo_w"]
                inner = bxb[:, hn:hn + qbx["h"], hw:hw + qbx["w"]]
                tag = f"rank {rank} {shape_a} {ga}->{gb} transport {transport}"
                assert torch.equal(inner, _dense(qbx, Y)), f"{tag}: interior"
                mask = torch.ones(bxb.shape[:3], dtype=torch.bool, device="cuda")
                mask[:, hn:hn + qbx["h"], hw:hw + qbx["w"]] = False
                assert bool((bxb[mask] == 5.0).all()), f"{tag}: margin written"
            dist.barrier()
            dc.dc_redist_destroy(r)
            dc.dc_plan_destroy(pb)
            dc.dc_plan_destroy(pa)
        dc.dc_comm_destroy(comm)
        dist.destroy_process_group()
    except Exception:
        errq.put(f"rank {rank}: {traceback.format_exc()}")
        raise


@pytest.mark.gpu
@pytest.mark.multigpu
@pytest.mark.parametrize("world", [2, 4])
def test_multigpu_redistribute(world):
    """Real ranks: the P2P all-to-all over CUDA-IPC peer memory and the NCCL
    send/recv transport leave every interior bitwise equal to the global
    tensor and the margins untouched (sample -> spatial, W -> H, 4-rank
    hybrid grids)."""
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
