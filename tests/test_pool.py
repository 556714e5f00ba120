"""Max pooling on the decomposition ("Pooling layers are
parallelized similarly", "halo exchanges before ... pooling";
SURVEY.md 8(f) NEXT-1): dc_pool_*.

GPU (1 GPU and loopback groups of 2-4 virtual ranks): forward with the x halo
exchange, backward with the dy halo exchange and the first maximum of every
window recomputed from the wide x halo; every rank's y is BITWISE the fp64
oracle's (oracle/network.py maxpool_fwd: a max copies a bf16 value exactly),
every dx within one bf16 rounding of the oracle's (a sum of <= ceil(K/S)^2
bf16 gradients, exact in fp32, rounded once)."""
import numpy as np
import pytest
import torch

import datagen
from oracle import network as net
from tests.gpu_util import fill_owned_only


@pytest.fixture(scope="module")
def dc():
    from paper_1903_06681_b200 import build
    build.build()
    import paper_1903_06681_b200 as dc
    return dc


def test_pool_errors(dc):
    with pytest.raises(dc.DCError):   # fp32
        dc.dc_pool_create(1, 16, 8, 8, 3, 2, 1, (1, 1, 1), dc.DC_FP32_3XTF32)
    with pytest.raises(dc.DCError):   # the model cannot pick a pooling grid
        dc.dc_pool_create(1, 16, 8, 8, 3, 2, 1, (0, 1, 1))
    with pytest.raises(dc.DCError):   # pad >= K
        dc.dc_pool_create(1, 16, 8, 8, 3, 2, 3, (1, 1, 1))
    with pytest.raises(dc.DCError):   # even windows (the conv geometry's odd-K reading)
        dc.dc_pool_create(1, 16, 8, 8, 2, 2, 0, (1, 1, 1))


CASES = [  # (N, C, H, W, K, S, P), grid
    ((2, 64, 24, 20, 3, 2, 1), (1, 1, 1)),    # ResNet's stem pool
    ((2, 64, 24, 20, 3, 2, 1), (1, 2, 1)),
    ((2, 64, 24, 20, 3, 2, 1), (1, 1, 2)),
    ((2, 64, 24, 20, 3, 2, 1), (1, 2, 2)),    # 2D grid: corners
    ((2, 32, 25, 23, 3, 2, 1), (2, 2, 1)),    # ragged, hybrid sample x spatial
    ((1, 16, 33, 17, 3, 2, 0), (1, 4, 1)),    # no padding, thin 4-way H split
    ((1, 16, 20, 18, 3, 1, 1), (1, 2, 1)),    # stride 1
]


@pytest.mark.gpu
@pytest.mark.parametrize("shape,grid", CASES)
def test_maxpool_parity(dc, shape, grid):
    N, C, H, W, K, S, P = shape
    Ho, Wo = (H + 2 * P - K) // S + 1, (W + 2 * P - K) // S + 1
    x = datagen.gen_x(N, C, H, W)
    # coarse values: many ties, so the first-maximum rule is exercised
    x = np.round(x * 4) / 4
    dy = datagen.gen_dy(N, C, Ho, Wo)
    y_ref, arg = net.maxpool_fwd(x, K, S, P)
    dx_ref = net.maxpool_bwd(dy, arg, H, W, K, S, P)
    world = grid[0] * grid[1] * grid[2]
    comms = dc.dc_comm_create_local(world, torch.cuda.current_device()) if world > 1 else [None]
    R = []
    try:
        for comm in comms:
            pool = dc.dc_pool_create(N, C, H, W, K, S, P, grid, dc.DC_BF16, comm)
            pin, pout = dc.dc_pool_plans(pool)
            qx, qy = dc.dc_plan_query(pin, dc.DC_X), dc.dc_plan_query(pout, dc.DC_Y)
            qdy, qdx = dc.dc_plan_query(pout, dc.DC_DY), dc.dc_plan_query(pout, dc.DC_DX)
            xb = dc.wrap_device_buffer(dc.dc_buffer_alloc(pin, dc.DC_X), (qx["n"], qx["hb"], qx["wb"], qx["c_pad"]))
            dyb = dc.wrap_device_buffer(dc.dc_buffer_alloc(pout, dc.DC_DY),
                                        (qdy["n"], qdy["hb"], qdy["wb"], qdy["c_pad"]))
            xb.copy_(fill_owned_only(x, qx))
            dyb.copy_(fill_owned_only(dy, qdy))
            stream = torch.cuda.ExternalStream(dc.dc_comm_stream(comm)) if comm else torch.cuda.current_stream()
            R.append(dict(pool=pool, qy=qy, qdx=qdx, xb=xb, dyb=dyb, s=stream,
                          y=torch.full((qy["n"], qy["h"], qy["w"], qy["c_pad"]), float("nan"), dtype=torch.bfloat16,
                                       device="cuda"),
                          dx=torch.full((qdx["n"], qdx["h"], qdx["w"], qdx["c_pad"]), float("nan"),
                                        dtype=torch.bfloat16, device="cuda")))
        torch.cuda.synchronize()
        for rep in range(2):    # twice: the halo epochs advance
            for d in R:
                with torch.cuda.stream(d["s"]):
                    dc.dc_pool_fwd(d["pool"], d["xb"], d["y"], dc.DC_EXCHANGE, d["s"])
                    dc.dc_pool_bwd(d["pool"], d["xb"], d["dyb"], d["dx"], dc.DC_EXCHANGE, d["s"])
            torch.cuda.synchronize()
            for r, d in enumerate(R):
                qy, qdx = d["qy"], d["qdx"]
                got = d["y"][..., :C].double().cpu().numpy().transpose(0, 3, 1, 2)
                ref = y_ref[qy["n0"]:qy["n0"] + qy["n"], :, qy["h0"]:qy["h0"] + qy["h"], qy["w0"]:qy["w0"] + qy["w"]]
                assert np.array_equal(got, ref), f"rank {r} rep {rep}: y differs"
                got = d["dx"][..., :C].double().cpu().numpy().transpose(0, 3, 1, 2)
                ref = dx_ref[qdx["n0"]:qdx["n0"] + qdx["n"], :, qdx["h0"]:qdx["h0"] + qdx["h"],
                             qdx["w0"]:qdx["w0"] + qdx["w"]]
                assert np.isfinite(got).all()
                assert (np.abs(got - ref) <= 2.0 ** -8 * np.abs(ref) + 1e-30).all(), f"rank {r} rep {rep}: dx"
    finally:
        for d in R:
            dc.dc_pool_destroy(d["pool"])
        for c in comms:
            if c is not None:
                dc.dc_comm_destroy(c)


@pytest.mark.gpu
@pytest.mark.parametrize("grid", [(1, 1, 1), (1, 2, 1), (1, 2, 2)])
def test_resnet_stem_chain(dc, grid):
    """ResNet's stem on the decomposition: conv 7x7/2 with
    the x halo exchange -> spatial BN statistics -> BN apply + ReLU written
    straight into the pooling's wide-halo input buffer (dst_plan = the
    pooling's in_plan) -> 3x3/2 max pool with its halo exchange, and the
    pooling backward. The pooled y is bitwise the oracle's max pool of the
    activation the ranks hold; dx within one bf16 rounding."""
    N, C, H, W, F = 2, 3, 48, 40, 64
    conv = (N, C, H, W, F, 7, 2, 3)
    Ha, Wa = 24, 20
    Hp, Wp = 12, 10
    x, w = datagen.gen_x(N, C, H, W), datagen.gen_w(F, C, 7)
    dyp = datagen.gen_dy(N, F, Hp, Wp)
    gam = torch.tensor(datagen.gen_block((1, F, 1, 1), 5, 11).ravel() + 1.25, dtype=torch.float32, device="cuda")
    bet = torch.tensor(datagen.gen_block((1, F, 1, 1), 5, 12).ravel() * 0.5, dtype=torch.float32, device="cuda")
    world = grid[0] * grid[1] * grid[2]
    comms = dc.dc_comm_create_local(world, torch.cuda.current_device()) if world > 1 else [None]
    R = []
    try:
        for comm in comms:
            pa = dc.dc_plan_create(*conv, grid, dc.DC_BF16, comm)
            pool = dc.dc_pool_create(N, F, Ha, Wa, 3, 2, 1, grid, dc.DC_BF16, comm)
            pin, pout = dc.dc_pool_plans(pool)
            qx, qy = dc.dc_plan_query(pa, dc.DC_X), dc.dc_plan_query(pa, dc.DC_Y)
            qpx, qpy = dc.dc_plan_query(pin, dc.DC_X), dc.dc_plan_query(pout, dc.DC_Y)
            qpdy, qpdx = dc.dc_plan_query(pout, dc.DC_DY), dc.dc_plan_query(pout, dc.DC_DX)
            xb = dc.wrap_device_buffer(dc.dc_buffer_alloc(pa, dc.DC_X), (qx["n"], qx["hb"], qx["wb"], qx["c_pad"]))
            pxb = dc.wrap_device_buffer(dc.dc_buffer_alloc(pin, dc.DC_X),
                                        (qpx["n"], qpx["hb"], qpx["wb"], qpx["c_pad"]))
            pdyb = dc.wrap_device_buffer(dc.dc_buffer_alloc(pout, dc.DC_DY),
                                         (qpdy["n"], qpdy["hb"], qpdy["wb"], qpdy["c_pad"]))
            xb.copy_(fill_owned_only(x, qx))
            pdyb.copy_(fill_owned_only(dyp, qpdy))
            wb = torch.zeros((F, 7, 7, qx["c_pad"]), dtype=torch.bfloat16, device="cuda")
            wb[..., :C] = torch.tensor(w.transpose(0, 2, 3, 1), dtype=torch.bfloat16)
            stream = torch.cuda.ExternalStream(dc.dc_comm_stream(comm)) if comm else torch.cuda.current_stream()
            R.append(dict(pa=pa, pool=pool, qpx=qpx, qpy=qpy, qpdx=qpdx, xb=xb, pxb=pxb, pdyb=pdyb, wb=wb, s=stream,
                          y=torch.empty((qy["n"], qy["h"], qy["w"], qy["c_pad"]), dtype=torch.bfloat16, device="cuda"),
                          yp=torch.empty((qpy["n"], qpy["h"], qpy["w"], qpy["c_pad"]), dtype=torch.bfloat16,
                                         device="cuda"),
                          dxp=torch.empty((qpdx["n"], qpdx["h"], qpdx["w"], qpdx["c_pad"]), dtype=torch.bfloat16,
                                          device="cuda"),
                          m=torch.zeros(F, dtype=torch.float64, device="cuda"),
                          v=torch.zeros(F, dtype=torch.float64, device="cuda")))
        torch.cuda.synchronize()
        for d in R:
            with torch.cuda.stream(d["s"]):
                dc.dc_conv_fwd(d["pa"], d["xb"].data_ptr(), d["wb"], d["y"], dc.DC_EXCHANGE | dc.DC_BN_STATS, d["s"])
                dc.dc_bn_spatial_stats(d["pa"], d["y"], d["m"], d["v"], dc.DC_BN_FROM_FWD, d["s"])
                pin, _ = dc.dc_pool_plans(d["pool"])
                dc.dc_bn_apply(d["pa"], d["y"], d["m"], d["v"], gam, bet, 1e-5, None, dc.DC_RELU, pin,
                               d["pxb"].data_ptr(), d["s"])
                dc.dc_pool_fwd(d["pool"], d["pxb"], d["yp"], dc.DC_EXCHANGE, d["s"])
                dc.dc_pool_bwd(d["pool"], d["pxb"], d["pdyb"], d["dxp"], dc.DC_EXCHANGE, d["s"])
        torch.cuda.synchronize()
        # the activation the ranks hold (owned blocks of the pooling inputs), global
        act = np.zeros((N, F, Ha, Wa))
        for d in R:
            q = d["qpx"]
            blk = d["pxb"][:, q["halo_n"]:q["halo_n"] + q["h"], q["halo_w"]:q["halo_w"] + q["w"], :F]
            act[q["n0"]:q["n0"] + q["n"], :, q["h0"]:q["h0"] + q["h"], q["w0"]:q["w0"] + q["w"]] = \
                blk.double().cpu().numpy().transpose(0, 3, 1, 2)
        assert (act >= 0).all() and (act > 0).any()            # ReLU'd, not empty
        y_ref, arg = net.maxpool_fwd(act, 3, 2, 1)
        dx_ref = net.maxpool_bwd(dyp, arg, Ha, Wa, 3, 2, 1)
        for r, d in enumerate(R):
            q = d["qpy"]
            got = d["yp"][..., :F].double().cpu().numpy().transpose(0, 3, 1, 2)
            assert np.array_equal(got, y_ref[q["n0"]:q["n0"] + q["n"], :, q["h0"]:q["h0"] + q["h"],
                                             q["w0"]:q["w0"] + q["w"]]), f"rank {r}: pooled y"
            q = d["qpdx"]
            got = d["dxp"][..., :F].double().cpu().numpy().transpose(0, 3, 1, 2)
            ref = dx_ref[q["n0"]:q["n0"] + q["n"], :, q["h0"]:q["h0"] + q["h"], q["w0"]:q["w0"] + q["w"]]
            assert (np.abs(got - ref) <= 2.0 ** -8 * np.abs(ref) + 1e-30).all(), f"rank {r}: pooling dx"
    finally:
        for d in R:
            dc.dc_pool_destroy(d["pool"])
            dc.dc_plan_destroy(d["pa"])
        for c in comms:
            if c is not None:
                dc.dc_comm_destroy(c)
