"""Multi-rank device protocols on ONE GPU (loopback group, dc_comm_create_local):
2-8 virtual ranks of this process, each with its own plan, margined buffers
and stream, exchange halos through the same P2P kernel and flag protocol the
real ranks use (plain device pointers in place of IPC-mapped peer memory).
This puts under the 1-GPU GPU test run:
  * the direct P2P halo exchange of x and dy: bit-exact;
  * the forward's interior -> boundary two-stream path with DC_EXCHANGE
     and the backward's dy exchange || filter gradient
    (PAPER.md:143): y and dx BITWISE equal to the 1-GPU plan with default
    settings (north_star), dW partials summing to the oracle's dW;
  * the spatial BN statistics over each rank group's NVLink mailbox
    (PAPER.md:149), fused-epilogue and separate-pass variants, vs the oracle;
  * CUDA-graph replay of every rank's step (device epochs stay in step);
  * the grid-agreement check and the NCCL-only transports' errors.
The NCCL transports (send/recv halo baseline, dW allreduce) are covered by
tests/test_multigpu*.py on 2 and 4 GPUs."""
import numpy as np
import pytest
import torch

import datagen
import oracle
from tests.gpu_util import (dw_to_fckk, fill_buffer, fill_owned_only, owned_nchw, rel_max, weights_gpu)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dc():
    from paper_1903_06681_b200 import build
    build.build()
    import paper_1903_06681_b200 as dc
    torch.cuda.init()
    return dc


CASES = [  # (N, C, H, W, F, K, S, P), grid
    ((1, 2, 16, 16, 4, 3, 1, 1), (1, 2, 1)),        # C1 (BASELINE configs[0]), 2-way H
    ((2, 16, 24, 20, 32, 3, 1, 1), (1, 1, 2)),      # W split: strided slabs
    ((2, 16, 24, 20, 32, 3, 1, 1), (1, 2, 2)),      # 2D grid: 8 neighbours incl. corners
    ((2, 16, 24, 20, 32, 3, 1, 1), (2, 2, 1)),      # hybrid sample x spatial: two BN groups
    ((1, 3, 40, 36, 64, 7, 2, 3), (1, 2, 1)),       # conv1-like 7x7/2: asymmetric strided halos
    ((1, 18, 33, 35, 64, 3, 2, 1), (1, 1, 2)),      # mesh conv1_1-like, stride 2 W split
    ((1, 32, 40, 24, 48, 5, 1, 2), (1, 4, 1)),      # K=5, 4-way H (thin shards)
    ((2, 64, 16, 16, 64, 3, 1, 1), (1, 2, 2)),      # 64-channel 128B-swizzle tiles
    ((1, 64, 33, 30, 128, 3, 2, 1), (1, 2, 4)),     # 8 ranks, stride 2, 2D
    ((1, 128, 20, 22, 64, 1, 1, 0), (1, 2, 2)),     # 1x1: no halo at all
]


class Ranks:
    """One loopback group running one layer: per-rank plans, IPC-free margined
    buffers (dc_buffer_alloc), dense outputs and streams."""

    def __init__(self, dc, shape, grid):
        self.dc, self.shape, self.grid = dc, shape, grid
        N, C, H, W, F, K, S, P = shape
        self.world = grid[0] * grid[1] * grid[2]
        self.comms = dc.dc_comm_create_local(self.world, torch.cuda.current_device())
        self.r = []
        for rank, comm in enumerate(self.comms):
            plan = dc.dc_plan_create(N, C, H, W, F, K, S, P, grid, dc.DC_BF16, comm)
            q = {t: dc.dc_plan_query(plan, t) for t in (dc.DC_X, dc.DC_Y, dc.DC_DY, dc.DC_DX)}
            xd, dyd = q[dc.DC_X], q[dc.DC_DY]
            xb = dc.wrap_device_buffer(dc.dc_buffer_alloc(plan, dc.DC_X), (xd["n"], xd["hb"], xd["wb"], xd["c_pad"]))
            dyb = dc.wrap_device_buffer(dc.dc_buffer_alloc(plan, dc.DC_DY),
                                        (dyd["n"], dyd["hb"], dyd["wb"], dyd["c_pad"]))
            yd, dxd = q[dc.DC_Y], q[dc.DC_DX]
            self.r.append(dict(
                plan=plan, q=q, xb=xb, dyb=dyb, stream=torch.cuda.ExternalStream(dc.dc_comm_stream(comm)),
                y=torch.full((yd["n"], yd["h"], yd["w"], yd["c_pad"]), float("nan"), dtype=torch.bfloat16,
                             device="cuda"),
                dx=torch.full((dxd["n"], dxd["h"], dxd["w"], dxd["c_pad"]), float("nan"), dtype=torch.bfloat16,
                              device="cuda"),
                dw=torch.full((F, K, K, C), float("nan"), dtype=torch.float32, device="cuda"),
                mean=torch.zeros(F, dtype=torch.float64, device="cuda"),
                var=torch.zeros(F, dtype=torch.float64, device="cuda")))

    def load_owned(self, x, dy):
        dc = self.dc
        for d in self.r:
            d["xb"].copy_(fill_owned_only(x, d["q"][dc.DC_X]))
            d["dyb"].copy_(fill_owned_only(dy, d["q"][dc.DC_DY]))
        torch.cuda.synchronize()

    def each(self, fn):
        """fn(rank dict) issued for every rank on its own stream (host calls
        never block: the ranks' kernels rendezvous on the device)."""
        for d in self.r:
            with torch.cuda.stream(d["stream"]):
                fn(d)
        torch.cuda.synchronize()

    def close(self):
        for d in self.r:
            self.dc.dc_plan_destroy(d["plan"])
        for c in self.comms:
            self.dc.dc_comm_destroy(c)


def reference(dc, shape, x, w, dy):
    """1-GPU plan, default settings: y, dx, dW of the whole layer."""
    N, C, H, W, F, K, S, P = shape
    plan = dc.dc_plan_create_virtual(N, C, H, W, F, K, S, P, (1, 1, 1), 0)
    try:
        xd, yd = dc.dc_plan_query(plan, dc.DC_X), dc.dc_plan_query(plan, dc.DC_Y)
        dyd, dxd = dc.dc_plan_query(plan, dc.DC_DY), dc.dc_plan_query(plan, dc.DC_DX)
        wb = weights_gpu(w, xd["c_pad"])
        Y = torch.empty((yd["n"], yd["h"], yd["w"], yd["c_pad"]), dtype=torch.bfloat16, device="cuda")
        DX = torch.empty((dxd["n"], dxd["h"], dxd["w"], dxd["c_pad"]), dtype=torch.bfloat16, device="cuda")
        DW = torch.empty((F, K, K, C), dtype=torch.float32, device="cuda")
        xr, dyr = fill_buffer(x, xd), fill_buffer(dy, dyd)
        dc.dc_conv_fwd(plan, xr, wb, Y, 0)
        dc.dc_conv_bwd_data(plan, dyr, wb, DX, 0)
        dc.dc_conv_bwd_filter(plan, xr, dyr, DW, 0)
        torch.cuda.synchronize()
        return wb, Y, DX, DW
    finally:
        dc.dc_plan_destroy(plan)


def inputs(shape):
    N, C, H, W, F, K, S, P = shape
    Ho, Wo = oracle.out_extent(H, K, S, P), oracle.out_extent(W, K, S, P)
    return datagen.gen_x(N, C, H, W), datagen.gen_w(F, C, K), datagen.gen_dy(N, F, Ho, Wo)


def owned_of(T, d):
    return T[d["n0"]:d["n0"] + d["n"], d["h0"]:d["h0"] + d["h"], d["w0"]:d["w0"] + d["w"]]


@pytest.mark.parametrize("shape,grid", CASES)
def test_loopback_halo_exchange_bitexact(dc, shape, grid):
    """dc_halo_exchange of x and dy between virtual ranks: every margined buffer
    (owned block + margins) equals the global tensor's window bit for bit, the
    positions outside the global tensor stay zero (never sent); twice in a row
    (the device epochs advance)."""
    x, _, dy = inputs(shape)
    R = Ranks(dc, shape, grid)
    try:
        for _ in range(2):
            R.load_owned(x, dy)
            R.each(lambda d: dc.dc_halo_exchange(d["plan"], dc.DC_X, d["xb"], 0, d["stream"]))
            R.each(lambda d: dc.dc_halo_exchange(d["plan"], dc.DC_DY, d["dyb"], 0, d["stream"]))
            for rank, d in enumerate(R.r):
                assert torch.equal(d["xb"], fill_buffer(x, d["q"][dc.DC_X])), f"rank {rank}: x margins"
                assert torch.equal(d["dyb"], fill_buffer(dy, d["q"][dc.DC_DY])), f"rank {rank}: dy margins"
    finally:
        R.close()


@pytest.mark.parametrize("shape,grid", CASES)
def test_loopback_overlapped_fwd_bwd_bitwise(dc, shape, grid):
    """The paper's overlapped layer on virtual ranks: forward with DC_EXCHANGE
    (x exchange on the comm stream || interior tiles, then boundary tiles,
    PAPER.md:177) and dc_conv_bwd with DC_EXCHANGE (dy exchange || filter
    gradient, then data gradient): every rank's y and dx are
    bitwise the default 1-GPU plan's; the rank-ordered sum of the local dW
    equals the 1-GPU dW within the fp32 bar and the oracle's dW."""
    N, C, H, W, F, K, S, P = shape
    x, w, dy = inputs(shape)
    wb, Y, DX, DW = reference(dc, shape, x, w, dy)
    R = Ranks(dc, shape, grid)
    try:
        R.load_owned(x, dy)
        R.each(lambda d: dc.dc_conv_fwd(d["plan"], d["xb"].data_ptr(), wb, d["y"],
                                        dc.DC_EXCHANGE | dc.DC_FORCE_OVERLAP, d["stream"]))
        R.each(lambda d: dc.dc_conv_bwd(d["plan"], d["xb"].data_ptr(), d["dyb"].data_ptr(), wb, d["dx"], d["dw"],
                                        dc.DC_EXCHANGE, d["stream"]))
        dw_sum = torch.zeros_like(DW)
        for rank, d in enumerate(R.r):
            q = d["q"]
            assert torch.equal(d["y"], owned_of(Y, q[dc.DC_Y])), f"rank {rank}: y not bitwise equal to 1 GPU"
            assert torch.equal(d["dx"], owned_of(DX, q[dc.DC_DX])), f"rank {rank}: dx not bitwise equal to 1 GPU"
            assert torch.equal(d["xb"], fill_buffer(x, q[dc.DC_X])), f"rank {rank}: x halo"
            assert torch.equal(d["dyb"], fill_buffer(dy, q[dc.DC_DY])), f"rank {rank}: dy halo"
            dw_sum += d["dw"]
        torch.cuda.synchronize()
        assert rel_max(dw_to_fckk(dw_sum, C), dw_to_fckk(DW, C)) <= 1e-4
        assert rel_max(dw_to_fckk(dw_sum, C), oracle.conv_bwd_filter(x, dy, K, S, P)) <= 1e-4
    finally:
        R.close()


def bn_bound(yn, depth):
    """fp32 groups (depth adds) then fp64; per channel."""
    u = 2.0 ** -24
    tm = depth * u * np.abs(yn).mean(axis=(0, 2, 3)) + 1e-12
    tv = depth * u * (yn * yn).mean(axis=(0, 2, 3)) + 2 * np.abs(yn.mean(axis=(0, 2, 3))) * tm + 1e-12
    return tm, tv


@pytest.mark.parametrize("shape,grid", [CASES[0], CASES[2], CASES[3], CASES[7], CASES[8]])
@pytest.mark.parametrize("fused", [False, True])
def test_loopback_spatial_bn_mailbox(dc, shape, grid, fused):
    """Spatially aggregated BN statistics (reading R11) through
    each BN group's one-shot mailbox: every rank of group i_N gets the mean and
    biased variance of the 1-GPU y over the group's samples and the WHOLE
    spatial extent, within the derived bound (both sides fp32 groups + fp64);
    with DC_BN_STATS + DC_BN_FROM_FWD the partials come from the forward
    epilogue. Twice in a row (mailbox parities alternate)."""
    N, C, H, W, F, K, S, P = shape
    x, w, dy = inputs(shape)
    wb, Y, _, _ = reference(dc, shape, x, w, dy)
    R = Ranks(dc, shape, grid)
    try:
        R.load_owned(x, dy)
        for _ in range(2):
            ff = dc.DC_EXCHANGE | (dc.DC_BN_STATS if fused else 0)
            R.each(lambda d: dc.dc_conv_fwd(d["plan"], d["xb"].data_ptr(), wb, d["y"], ff, d["stream"]))
            bf = dc.DC_BN_FROM_FWD if fused else 0
            R.each(lambda d: dc.dc_bn_spatial_stats(d["plan"], d["y"], d["mean"], d["var"], bf, d["stream"]))
            for rank, d in enumerate(R.r):
                yd = d["q"][dc.DC_Y]
                yn = Y[yd["n0"]:yd["n0"] + yd["n"], ..., :F].permute(0, 3, 1, 2).double().cpu().numpy()
                m_ref, v_ref = oracle.bn_stats(yn)
                tm, tv = bn_bound(yn, 2 * 40)
                assert (np.abs(d["mean"].cpu().numpy() - m_ref) <= tm).all(), f"rank {rank} mean"
                assert (np.abs(d["var"].cpu().numpy() - v_ref) <= tv).all(), f"rank {rank} var"
    finally:
        R.close()


@pytest.mark.parametrize("shape,grid", [CASES[2], CASES[4], CASES[8]])
def test_loopback_graph_replay(dc, shape, grid):
    """Each virtual rank's layer step (fwd with exchange + fused BN, spatial BN,
    overlapped bwd) captured once into a CUDA graph on its own stream and
    replayed 3 times concurrently with the other ranks' graphs: the
    device-side epochs of the halo and BN protocols keep the ranks in step and
    every replay reproduces the eager results bit for bit."""
    N, C, H, W, F, K, S, P = shape
    x, w, dy = inputs(shape)
    wb, Y, DX, _ = reference(dc, shape, x, w, dy)
    R = Ranks(dc, shape, grid)
    try:
        R.load_owned(x, dy)

        def step(d):
            dc.dc_conv_fwd(d["plan"], d["xb"].data_ptr(), wb, d["y"], dc.DC_EXCHANGE | dc.DC_BN_STATS, d["stream"])
            dc.dc_bn_spatial_stats(d["plan"], d["y"], d["mean"], d["var"], dc.DC_BN_FROM_FWD, d["stream"])
            dc.dc_conv_bwd(d["plan"], d["xb"].data_ptr(), d["dyb"].data_ptr(), wb, d["dx"], d["dw"],
                           dc.DC_EXCHANGE, d["stream"])

        R.each(step)  # eager (also warms up)
        eager = [(d["y"].clone(), d["dx"].clone(), d["dw"].clone(), d["mean"].clone(), d["var"].clone())
                 for d in R.r]
        graphs = []
        for d in R.r:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=d["stream"], capture_error_mode="thread_local"):
                step(d)
            graphs.append(g)
        torch.cuda.synchronize()
        for _ in range(3):
            for d in R.r:
                d["y"].fill_(float("nan"))
                d["dx"].fill_(float("nan"))
            torch.cuda.synchronize()
            for d, g in zip(R.r, graphs):
                with torch.cuda.stream(d["stream"]):
                    g.replay()
            torch.cuda.synchronize()
            for rank, (d, e) in enumerate(zip(R.r, eager)):
                assert torch.equal(d["y"], e[0]) and torch.equal(d["y"], owned_of(Y, d["q"][dc.DC_Y])), rank
                assert torch.equal(d["dx"], e[1]) and torch.equal(d["dx"], owned_of(DX, d["q"][dc.DC_DX])), rank
                assert torch.equal(d["dw"], e[2]), f"rank {rank}: dW differs between replays"
                assert torch.equal(d["mean"], e[3]) and torch.equal(d["var"], e[4]), rank
        del graphs
    finally:
        R.close()


def test_loopback_nccl_transports_and_grid_agreement(dc):
    """NCCL-only transports fail loudly in a loopback group; ranks whose
    performance models pick different grids are rejected at plan creation
    (instead of building mismatched neighbour lists)."""
    shape, grid = CASES[0]
    N, C, H, W, F, K, S, P = shape
    R = Ranks(dc, shape, grid)
    try:
        d = R.r[0]
        with pytest.raises(dc.DCError) as e:
            dc.dc_halo_exchange(d["plan"], dc.DC_X, d["xb"], dc.DC_HALO_NCCL)
        assert e.value.status == dc.DC_ERR_UNSUPPORTED
        with pytest.raises(dc.DCError) as e:
            dc.dc_conv_bwd_filter(d["plan"], d["xb"].data_ptr(), d["dyb"].data_ptr(), d["dw"], dc.DC_ALLREDUCE)
        assert e.value.status == dc.DC_ERR_UNSUPPORTED
    finally:
        R.close()
    # a wide, short layer: an H split sends O*C*W_l words, a W split O*C*H_l;
    # with exposed halos (overlap off) a pure bandwidth model picks the W split,
    # a large extra latency on strided (W-split) messages picks the H split
    L = (1, 64, 64, 1024, 64, 3, 1, 1)
    comms = dc.dc_comm_create_local(2, torch.cuda.current_device())
    plans = []
    try:
        dc.dc_model_set_overlap(False)
        dc.dc_model_set_comm(1e-6, 1e-9)
        dc.dc_model_set_strided_latency(0.0)
        plans.append(dc.dc_plan_create(*L, (1, 0, 0), dc.DC_BF16, comms[0]))
        assert dc.dc_plan_decomp(plans[0])[0] == (1, 1, 2)
        dc.dc_model_set_strided_latency(1.0)
        assert dc.dc_model_choose_fixed(*L, 2, (1, 0, 0))[0] == (1, 2, 1)
        with pytest.raises(dc.DCError) as e:
            plans.append(dc.dc_plan_create(*L, (1, 0, 0), dc.DC_BF16, comms[1]))
        assert e.value.status == dc.DC_ERR_PARTITION
    finally:
        dc.dc_model_set_overlap(True)
        dc.dc_model_set_comm(5e-6, 1 / 700e9)
        dc.dc_model_set_strided_latency(0.0)
        for p in plans:
            dc.dc_plan_destroy(p)
        for c in comms:
            dc.dc_comm_destroy(c)
