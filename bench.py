"""bench.py -- conv fwd+bwd time & TFLOP/s (% peak) of the spatially / hybrid
partitioned convolution hot path (arXiv:1903.06681) on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME]
  torchrun --nproc-per-node N bench.py --gpus N ...        (one rank per GPU)
  python bench.py --impl reference ...                      (fp64 CPU oracle arm)

One step = for every layer of the workload: forward (with x halo exchange
overlapped with interior tiles), spatially aggregated BN statistics of its
output, and backward (dy halo || filter gradient, then data gradient || dW
allreduce), i.e. every row of SURVEY.md 8(a) on the hot path, through the C
ABI (libdconv.so); the decomposition of every layer comes from the library's
performance model (a8) unless --decomp is given. Global batch fixed as N grows
(strong scaling). Default workload: the 2K mesh-tangling conv stack at N = 8
(BASELINE.json configs[3], "N=1-8, pure spatial decomposition"), every layer
on the pure spatial grid (1, pH, pW) the library's performance model picks
(PAPER.md:218-226); --decomp auto lets it use sample parallelism too.
Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

# the library's side streams (dconv.h: dc_comm_create) on distinct hardware
# queues: set before CUDA initialises (the runtime's default is 8)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# (name, N, C, H, W, F, K, S, P)
def mesh_stack(size: int = 2048, n: int = 1, blocks: int = 6, per_block: int = 5):
    """The mesh-tangling CNN's conv stack: six blocks of three
    (1K) or five (2K) 3x3 convolutions, the first of each block stride 2, and
    a final prediction conv. The widths are not in the paper (lost figures):
    DESIGN.md reading R20 (F = 64, 128, 256, 512, 512, 512; final 1x1 -> 2)."""
    widths = [64, 128, 256, 512, 512, 512][:blocks]
    layers, c, h = [], 18, size
    for b, f in enumerate(widths, 1):
        for k in range(1, per_block + 1):
            s = 2 if k == 1 else 1
            layers.append((f"conv{b}_{k}", n, c, h, h, f, 3, s, 1))
            h = (h + 2 - 3) // s + 1
            c = f
    layers.append(("pred", n, c, h, h, 2, 1, 1, 0))
    return layers


def resnet50_convs(n: int = 64, size: int = 224):
    """The 53 convolutions of ResNet-50 with Caffe's
    stride placement (stride 2 in branch2a 1x1 and branch1, reading R21):
    conv1 7x7/2, then 3/4/6/3 bottleneck blocks (1x1, 3x3, 1x1; projection
    branch1 in the first block of each stage). The conv-stack proxy of
    BASELINE.json configs[2] (pooling, BN apply, ReLU, residual adds and the FC
    layer are not convolutions: NEXT-1)."""
    layers = [("conv1", n, 3, size, size, 64, 7, 2, 3)]
    h, c = size // 4, 64  # after conv1 (/2) and the 3x3/2 max-pool (/2)
    for stage, (blocks, mid, out) in enumerate([(3, 64, 256), (4, 128, 512), (6, 256, 1024), (3, 512, 2048)], 2):
        for b in range(blocks):
            tag = f"res{stage}{chr(ord('a') + b)}"
            s = 2 if (b == 0 and stage > 2) else 1
            if b == 0:
                layers.append((f"{tag}_branch1", n, c, h, h, out, 1, s, 0))
            layers.append((f"{tag}_branch2a", n, c, h, h, mid, 1, s, 0))
            h2 = (h - 1) // s + 1
            layers.append((f"{tag}_branch2b", n, mid, h2, h2, mid, 3, 1, 1))
            layers.append((f"{tag}_branch2c", n, mid, h2, h2, out, 1, 1, 0))
            h, c = h2, out
    return layers


WORKLOADS = {
    # BASELINE.json configs[3]: 2K mesh-tangling CNN conv stack, N = 1-8, pure
    # spatial strong scaling. Default: N = 8 (a global mini-batch fixed as the
    # GPUs grow); N = 1 is the latency-bound end of the same config.
    "mesh2k_n8": mesh_stack(2048, 8),
    "mesh2k": mesh_stack(2048, 1),
    "mesh1k": mesh_stack(1024, 1, per_block=3),
    # BASELINE.json configs[3], end to end (NEXT-1): the same stack as ONE
    # network -- BN + ReLU between the convolutions, the backward chained
    # through them (NET_WORKLOADS below)
    "mesh2k_n8_net": mesh_stack(2048, 8),
    "mesh2k_net": mesh_stack(2048, 1),
    # BASELINE.json configs[2]: the 53 ResNet-50 convolutions at N = 64, 224^2
    "resnet50_n64": resnet50_convs(64),
    # BASELINE.json configs[1]: ResNet-50 conv layers at N=32, 224x224
    "resnet_layers": [("conv1", 32, 3, 224, 224, 64, 7, 2, 3),
                      ("res2a_branch2b", 32, 64, 56, 56, 64, 3, 1, 1),
                      ("res3b_branch2a", 32, 512, 28, 28, 128, 1, 1, 0)],
    # per-layer proxies of configs[3]
    "mesh2k_layers": [("conv1_1", 1, 18, 2048, 2048, 64, 3, 2, 1),
                      ("conv1_2", 1, 64, 1024, 1024, 64, 3, 1, 1)],
    # BASELINE.json configs[0]
    "c1": [("c1", 1, 2, 16, 16, 4, 3, 1, 1)],
}


NET_WORKLOADS = {"mesh2k_n8_net", "mesh2k_net"}


def layer_flops(l) -> float:
    """Algorithmic FLOPs of one conv op (fwd; bwd-data and bwd-filter are the
    same count): 2 N F C K^2 Ho Wo."""
    _, N, C, H, W, F, K, S, P = l
    Ho, Wo = (H + 2 * P - K) // S + 1, (W + 2 * P - K) // S + 1
    return 2.0 * N * F * C * K * K * Ho * Wo


def layer_bytes(l, op: str, e: int = 2) -> float:
    """Minimum HBM bytes of one conv op (activations and weights in/out once,
    e bytes per element: 2 bf16, 4 fp32; dW fp32)."""
    _, N, C, H, W, F, K, S, P = l
    Ho, Wo = (H + 2 * P - K) // S + 1, (W + 2 * P - K) // S + 1
    act = float(e) * (N * H * W * C + N * Ho * Wo * F)
    return act + (4.0 if op == "bpw" else float(e)) * F * C * K * K


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """SM clock + clock-event (throttle) reasons sampled every ~5 ms through
    NVML during the timed region (a 120 ms region still gets ~20 samples);
    nvidia-smi at 100 ms as the fallback. Field names differ across drivers:
    probe and fall back."""
    REASONS = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    VARIANTS = [",".join(["clocks.sm", "clocks.max.sm"] + [f"clocks_event_reasons.{r}" for r in REASONS]),
                ",".join(["clocks.sm", "clocks.max.sm"] + [f"clocks_throttle_reasons.{r}" for r in REASONS]),
                "clocks.sm,clocks.max.sm"]

    def __init__(self, gpu: int):
        self.gpu, self.proc, self.lines, self.q = gpu, None, [], None
        self.nvml, self.samples, self.stop_flag = None, [], threading.Event()

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            import torch
            pr = torch.cuda.get_device_properties(self.gpu)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.gpu)

    def start(self):
        try:
            nv, h = self._nvml_handle()
            bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))

            def poll():
                while not self.stop_flag.is_set():
                    try:
                        sm = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((sm, [n for n, b in bits.items() if r & b]))
                    except Exception:
                        pass
                    time.sleep(0.005)
            self.nvml = threading.Thread(target=poll, daemon=True)
            self.nvml.start()
            time.sleep(0.05)
            return
        except Exception:
            self.nvml = None
        for q in self.VARIANTS:
            try:
                r = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                    "--format=csv,noheader,nounits"],
                                   capture_output=True, text=True, timeout=20)
                if r.returncode == 0 and "," in r.stdout:
                    self.q = q
                    break
            except Exception:
                return
        if self.q is None:
            return
        self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.q}",
                                      "--format=csv,noheader,nounits", "-lms", "100"],
                                     stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        self.t = threading.Thread(target=lambda: self.lines.extend(iter(self.proc.stdout.readline, "")),
                                  daemon=True)
        self.t.start()
        time.sleep(0.3)

    def stop(self):
        if self.nvml is not None:
            self.stop_flag.set()
            self.nvml.join(timeout=2)
            sm = [s for s, _ in self.samples]
            reasons = sorted({n for _, rs in self.samples for n in rs})
            mx = self.max_mhz
            load = [v for v in sm if mx and v > 0.3 * mx] or sm
            return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx, "reasons": reasons,
                    "samples": len(sm), "fields": "NVML clocks (SM) + current clock-event reasons, 5 ms"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except (ValueError, IndexError):
                continue
            for n, v in zip(self.REASONS, f[2:]):
                if v.lower() == "active":
                    reasons.add(n)
        load = [s for s in sm if mx and s > 0.3 * mx] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm), "fields": self.q}


# ----------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline and --impl reference)
# ----------------------------------------------------------------------------
def oracle_sample(layers, budget_s: float = 15.0):
    """Times the fp64 oracle (as it stands) on a bounded sample of the
    workload: for every layer, Eq. 1 on its first output rows, on inputs
    generated only for the rows they read (the 2K-mesh tensors are never
    materialised on the host). fwd, bwd-data and bwd-filter have the same
    algorithmic FLOPs, so the rate transfers to the fwd+bwd metric.
    Returns (algorithmic FLOPs computed, seconds, description)."""
    import datagen
    import oracle
    flops = secs = 0.0
    desc = []
    per_layer = budget_s / len(layers)
    for l in layers:
        name, N, C, H, W, F, K, S, P = l
        Ho, Wo = (H + 2 * P - K) // S + 1, (W + 2 * P - K) // S + 1
        n = min(N, 2)
        row_flops = 2.0 * n * F * C * K * K * Wo
        rows = int(max(1, min(Ho, per_layer / (row_flops / (1e9 * oracle.num_threads())))))
        x = datagen.gen_x(N, C, H, W, n=(0, n), h=(0, min(H, S * rows - P + K)))
        w = datagen.gen_w(F, C, K)
        t0 = time.perf_counter()
        oracle.conv_fwd(x, w, S, P, rows=(0, rows))
        secs += time.perf_counter() - t0
        flops += row_flops * rows
        desc.append(f"{name}[n={n},rows 0-{rows}]")
    return flops, secs, "Eq.1 output rows of every layer: " + " ".join(desc)


def run_reference(args, layers, wl_name):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    oracle.build()
    steps = []
    for _ in range(args.warmup):
        oracle_sample(layers, budget_s=2.0)
    desc = ""
    for _ in range(args.steps):
        f, s, desc = oracle_sample(layers, budget_s=args.ref_budget)
        steps.append((f, s))
    flops = sum(f for f, _ in steps)
    secs = sum(s for _, s in steps)
    value = flops / secs / 1e12
    threads = oracle.num_threads()
    print(json.dumps({
        "impl": "reference", "metric": "conv fwd+bwd TFLOP/s", "value": value, "unit": "TFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * secs / max(1, args.steps), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl_name, "layers": [l[0] for l in layers], "global_batch": layers[0][1]},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads, "kind": "oracle",
                         "sample": desc},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), file=JSON_OUT, flush=True)


# ----------------------------------------------------------------------------
# GPU arm
# ----------------------------------------------------------------------------
def _claim_stdout():
    """The JSON line is the only thing bench.py writes to stdout: everything
    else that writes to fd 1 (NCCL's version banner at communicator init,
    library prints) is redirected to stderr; the line goes to a dup of the
    original stdout."""
    global JSON_OUT
    sys.stdout.flush()
    JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)


JSON_OUT = sys.stdout


def main():
    _claim_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="mesh2k_n8", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--decomp", default="spatial",
                    help="spatial (model picks pH x pW, pN = 1: BASELINE configs[3]) | auto (model, all grids) | "
                         "pn,ph,pw (0 entries: model's choice) | strategy (network workloads: the model's "
                         "parallel execution strategy, one grid per layer with redistributions between, "
                         "PAPER.md:216-228)")
    ap.add_argument("--halo", default="p2p", choices=["p2p", "nccl"])
    ap.add_argument("--no-overlap", action="store_true",
                    help="ablation: finish each halo exchange before the conv (DC_NO_OVERLAP)")
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp32"],
                    help="bf16: bf16 x bf16 -> fp32 (DC_BF16); fp32: the paper's single precision via 3xTF32 "
                         "(DC_FP32_3XTF32)")
    ap.add_argument("--splitk-basis", type=int, default=0,
                    help="dc_plan_set_splitk_world on every plan (0: the library's fixed basis; A/B only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-budget", type=float, default=8.0)
    ap.add_argument("--no-fused-bn", action="store_true", help="BN statistics by a separate pass over y")
    ap.add_argument("--ablate", default="", help="DIAGNOSTIC: comma list of exchange,bn,allreduce to skip")
    ap.add_argument("--ar-sync", action="store_true", help="join each dW allreduce inside its layer's call")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="replay the step as a CUDA graph")
    ap.add_argument("--cost-table-in", default=os.path.join(ROOT, "profiles", "cost_table_b200.csv"),
                    help="measured local conv costs for the performance model ('' = roofline estimate)")
    ap.add_argument("--cost-table", default=None, help="write the per-op timings as a cost table CSV")
    ap.add_argument("--watchdog", type=float, default=1500.0,
                    help="seconds after which a run that has not finished prints every thread's stack and exits")
    args = ap.parse_args()
    import faulthandler
    if args.watchdog > 0:
        faulthandler.dump_traceback_later(args.watchdog, exit=True)
    layers = WORKLOADS[args.workload]
    NET = args.workload in NET_WORKLOADS
    if args.impl == "reference":
        return run_reference(args, layers, args.workload)

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1903_06681_b200 import build
    build.build()
    import paper_1903_06681_b200 as dc
    import datagen

    fp32 = args.dtype == "fp32"
    DTYPE = dc.DC_FP32_3XTF32 if fp32 else dc.DC_BF16
    TDT = torch.float32 if fp32 else torch.bfloat16
    KIND = "act24" if fp32 else "act"          # fp32-exact 24-bit grid / bf16-exact grid
    IMPORT_SRC = 0 if fp32 else dc.DC_SRC_BF16  # the source's element type

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE {world}"
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        uid = [dc.dc_comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = dc.dc_comm_create(rank, world, uid[0], local)
    else:
        comm = dc.dc_comm_create(0, 1, None, local)
    stream = torch.cuda.Stream()
    sp = stream.cuda_stream
    halo_flag = dc.DC_HALO_NCCL if args.halo == "nccl" else 0
    # dW allreduces are queued on the communicator's gradient stream and joined
    # once at the end of the step (overlapped with later layers)
    FLAGS = dc.DC_EXCHANGE | dc.DC_ALLREDUCE | halo_flag | (0 if args.ar_sync else dc.DC_ALLREDUCE_ASYNC)
    if args.no_overlap:
        FLAGS |= dc.DC_NO_OVERLAP
    ablate = set(a for a in args.ablate.split(",") if a)  # diagnostics only: the JSON says so
    if "exchange" in ablate:
        FLAGS &= ~dc.DC_EXCHANGE
    if "allreduce" in ablate:
        FLAGS &= ~dc.DC_ALLREDUCE

    # the performance model's local conv costs: measured on B200 by
    # tools/calibrate.py, roofline fallback otherwise
    table = args.cost_table_in
    if table and os.path.exists(table):
        dc.dc_model_load_table(table)
    else:
        table = None
    # communication terms fitted to this implementation on B200:
    # the exposed cost of one halo message (handshake + boundary tiles), strided
    # east/west messages dearer, exchanges charged without overlap (measured:
    # not hidden, profiles/r1_NOTES.md)
    MODEL_COMM = {"alpha_s": 13e-6, "beta_s_per_byte": 1 / 700e9, "alpha_strided_extra_s": 6e-6, "overlap": False}
    dc.dc_model_set_comm(MODEL_COMM["alpha_s"], MODEL_COMM["beta_s_per_byte"])
    dc.dc_model_set_strided_latency(MODEL_COMM["alpha_strided_extra_s"])
    dc.dc_model_set_overlap(MODEL_COMM["overlap"])
    # ---- one grid for a whole network (its layers hand activations over in
    # place): the pure spatial grid with the least total model cost over the
    # layers (PAPER.md:218-226 with no redistribution between layers) ----
    net_grid = None
    strategy = None
    if args.decomp == "strategy":
        if not NET:
            raise SystemExit("--decomp strategy needs a network workload (*_net)")
        # one grid per layer: the shortest path over the per-layer candidates
        # with Shuffle edges (chain: parent = previous layer)
        chain = [tuple(l[1:]) + (i - 1,) for i, l in enumerate(layers)]
        sgrids, stotal = dc.dc_model_strategy(chain, world)
        strategy = {"grids": [list(g) for g in sgrids], "model_step_ms": stotal * 1e3}
    elif NET:
        if args.decomp in ("auto", "spatial"):
            best = None
            for ph in range(world, 0, -1):
                if world % ph:
                    continue
                g = (1, ph, world // ph)
                try:
                    t = sum(dc.dc_model_layer_cost(*l[1:], g) for l in layers)
                except dc.DCError:
                    continue  # invalid for some layer
                if best is None or t < best[0]:
                    best = (t, g)
            net_grid = best[1]
        else:
            net_grid = tuple(int(v) for v in args.decomp.split(","))
    # ---- per-layer plans and resident inputs ----
    L = []
    for li, l in enumerate(layers):
        name, N, C, H, W, F, K, S, P = l
        if strategy:
            decomp = tuple(strategy["grids"][li])
        else:
            decomp = net_grid or {"auto": (0, 0, 0), "spatial": (1, 0, 0)}.get(args.decomp) or tuple(
                int(v) for v in args.decomp.split(","))
        plan = dc.dc_plan_create(N, C, H, W, F, K, S, P, decomp, DTYPE, comm)
        if args.splitk_basis:
            dc.dc_plan_set_splitk_world(plan, args.splitk_basis)
        chosen, pred = dc.dc_plan_decomp(plan)
        xd, yd = dc.dc_plan_query(plan, dc.DC_X), dc.dc_plan_query(plan, dc.DC_Y)
        dyd, dxd = dc.dc_plan_query(plan, dc.DC_DY), dc.dc_plan_query(plan, dc.DC_DX)
        wd = dc.dc_plan_query(plan, dc.DC_W)
        xb = dc.wrap_device_buffer(dc.dc_buffer_alloc(plan, dc.DC_X), (xd["n"], xd["hb"], xd["wb"], xd["c_pad"]),
                                   TDT)
        dyb = dc.wrap_device_buffer(dc.dc_buffer_alloc(plan, dc.DC_DY),
                                    (dyd["n"], dyd["hb"], dyd["wb"], dyd["c_pad"]), TDT)

        def owned(desc, tid, shape, ch):
            # the counter-based generator run on the GPU (bitwise equal to the
            # numpy one, tests/test_datagen.py): no host hashing of gigabytes;
            # the owned block, dense, logical channels (dc_tensor_import's source)
            return datagen.gen_block_nhwc_torch(
                shape, datagen.SEED, tid, kind=KIND, n=(desc["n0"], desc["n0"] + desc["n"]),
                h=(desc["h0"], desc["h0"] + desc["h"]), w=(desc["w0"], desc["w0"] + desc["w"]),
                c_pad=ch, dtype=TDT, device="cuda")

        Ho, Wo = (H + 2 * P - K) // S + 1, (W + 2 * P - K) // S + 1
        x_own = owned(xd, datagen.TID_X, (N, C, H, W), C)
        dy_own = owned(dyd, datagen.TID_DY, (N, F, Ho, Wo), F)
        # into the margined buffers through the C ABI (fp32 plans: the 3xTF32 split)
        dc.dc_tensor_import(plan, dc.DC_X, x_own, xb, IMPORT_SRC)
        dc.dc_tensor_import(plan, dc.DC_DY, dy_own, dyb, IMPORT_SRC)
        wnp = np.zeros((F, K, K, wd["c_pad"]), dtype=np.float32)
        wnp[..., :C] = datagen.gen_w(F, C, K, kind=KIND).transpose(0, 2, 3, 1)
        wt = torch.tensor(wnp, dtype=TDT).cuda()
        y = torch.empty((yd["n"], yd["h"], yd["w"], yd["c_pad"]), dtype=TDT, device="cuda")
        dx = torch.empty((dxd["n"], dxd["h"], dxd["w"], dxd["c_pad"]), dtype=TDT, device="cuda")
        dw = torch.empty((F, K, K, C), dtype=torch.float32, device="cuda")
        bn_mean = torch.empty(F, dtype=torch.float64, device="cuda")
        bn_var = torch.empty(F, dtype=torch.float64, device="cuda")
        # BN scale / shift of the network workloads (and their gradients)
        gamma = torch.tensor(1.0 + 0.25 * datagen.gen_block((1, F, 1, 1), datagen.SEED, 7).ravel(),
                             dtype=torch.float32, device="cuda")
        beta = torch.tensor(0.1 * datagen.gen_block((1, F, 1, 1), datagen.SEED, 8).ravel(), dtype=torch.float32,
                            device="cuda")
        dgamma, dbeta = torch.empty_like(gamma), torch.empty_like(beta)
        # pinned host copies for the end-to-end leg (dense, logical channels)
        host = {"x": x_own.cpu().pin_memory(), "dy": dy_own.cpu().pin_memory(), "w": wt.cpu().pin_memory(),
                "dw": torch.empty(dw.shape, dtype=torch.float32).pin_memory()}
        L.append(dict(l=l, plan=plan, decomp=chosen, pred=pred, xd=xd, dyd=dyd, xb=xb, dyb=dyb, w=wt, y=y,
                      dx=dx, dw=dw, bn_mean=bn_mean, bn_var=bn_var, gamma=gamma, beta=beta, dgamma=dgamma,
                      dbeta=dbeta, host=host))
    # ---- redistributions where consecutive layers use different grids
    # (PAPER.md:151-153): forward the BN / ReLU output (dense, this layer's
    # grid) into the next layer's margined x; backward the next layer's dx
    # into this layer's dense BN-output gradient ----
    n_shuffles = 0
    if NET:
        for i in range(len(L) - 1):
            d, n = L[i], L[i + 1]
            if tuple(d["decomp"]) == tuple(n["decomp"]):
                continue
            yd = dc.dc_plan_query(d["plan"], dc.DC_Y)
            d["act"] = torch.empty((yd["n"], yd["h"], yd["w"], yd["c_pad"]), dtype=TDT, device="cuda")
            d["dout"] = dc.wrap_device_buffer(dc.dc_buffer_alloc(d["plan"], dc.DC_Y),
                                              (yd["n"], yd["h"], yd["w"], yd["c_pad"]), TDT)
            d["r_fwd"] = dc.dc_redist_create(d["plan"], dc.DC_Y, n["plan"], dc.DC_X)
            d["r_bwd"] = dc.dc_redist_create(n["plan"], dc.DC_DX, d["plan"], dc.DC_Y)
            n_shuffles += 1
    torch.cuda.synchronize()

    fused = not ("bn" in ablate or args.no_fused_bn)

    def conv_fwd_ops(i, d):
        """Forward of layer i: conv (+ fused BN partials) and the spatially
        aggregated BN statistics of its output."""
        fwd_flags = FLAGS | (dc.DC_BN_STATS if fused else 0)
        bn_flags = dc.DC_BN_FROM_FWD if fused else 0
        ops = [(i, "fwd", lambda: dc.dc_conv_fwd(d["plan"], d["xb"].data_ptr(), d["w"], d["y"], fwd_flags, sp))]
        if "bn" not in ablate:
            ops.append((i, "bn", lambda: dc.dc_bn_spatial_stats(d["plan"], d["y"], d["bn_mean"], d["bn_var"],
                                                                bn_flags, sp)))
        return ops

    def conv_bwd_ops(i, d):
        if world == 1:
            # no halo / allreduce at one rank: the two backward kernels are
            # called separately so each gets its own timing
            return [(i, "bpw", lambda: dc.dc_conv_bwd_filter(d["plan"], d["xb"].data_ptr(), d["dyb"].data_ptr(),
                                                             d["dw"], FLAGS, sp)),
                    (i, "bpx", lambda: dc.dc_conv_bwd_data(d["plan"], d["dyb"].data_ptr(), d["w"], d["dx"], FLAGS,
                                                           sp))]
        return [(i, "bwd", lambda: dc.dc_conv_bwd(d["plan"], d["xb"].data_ptr(), d["dyb"].data_ptr(), d["w"],
                                                  d["dx"], d["dw"], FLAGS, sp))]

    def step_ops():
        """The calls of one step in order: (layer, op name, fn).
        Conv-stack workloads: every layer forward and backward on its own
        resident inputs. Network workloads (NEXT-1): the forward chains
        conv -> BN statistics -> BN apply + ReLU straight into the next layer's
        margined input; the backward runs from the last layer down, each
        layer's dx going through the BN / ReLU backward (group sums over the
        spatial group) into the previous layer's margined dy."""
        ops = []
        if not NET:
            for i, d in enumerate(L):
                ops += conv_fwd_ops(i, d) + conv_bwd_ops(i, d)
            return ops
        for i, d in enumerate(L):
            ops += conv_fwd_ops(i, d)
            if i + 1 < len(L):
                n = L[i + 1]
                if "r_fwd" in d:  # a different grid next: BN / ReLU densely, then the shuffle
                    ops.append((i, "act", lambda d=d: dc.dc_bn_apply(
                        d["plan"], d["y"], d["bn_mean"], d["bn_var"], d["gamma"], d["beta"], 1e-5, None,
                        dc.DC_RELU, None, d["act"], sp)))
                    ops.append((i, "shuf", lambda d=d, n=n: dc.dc_redistribute(d["r_fwd"], d["act"], n["xb"], 0,
                                                                               sp)))
                    continue
                ops.append((i, "act", lambda d=d, n=n: dc.dc_bn_apply(
                    d["plan"], d["y"], d["bn_mean"], d["bn_var"], d["gamma"], d["beta"], 1e-5, None, dc.DC_RELU,
                    n["plan"], n["xb"].data_ptr(), sp)))
        for i in range(len(L) - 1, -1, -1):
            d = L[i]
            ops += conv_bwd_ops(i, d)
            if i > 0:
                p = L[i - 1]
                dout = d["dx"]
                if "r_bwd" in p:  # the gradient back onto the previous layer's grid
                    ops.append((i - 1, "shufb", lambda d=d, p=p: dc.dc_redistribute(p["r_bwd"], d["dx"], p["dout"],
                                                                                    0, sp)))
                    dout = p["dout"]
                ops.append((i - 1, "bnb", lambda d=d, p=p, dout=dout: dc.dc_bn_backward(
                    p["plan"], dout, p["y"], p["bn_mean"], p["bn_var"], p["gamma"], p["beta"],
                    p["dyb"].data_ptr(), 1e-5, None, dc.DC_RELU, p["dgamma"], p["dbeta"], None, sp)))
        return ops

    def step(e2e=False):
        if e2e:
            # inputs arrive from pinned HOST memory every step through the C ABI
            # (dc_tensor_import with host pointers): every layer's copies are
            # queued up front on the plans' copy streams, so they overlap the
            # compute of the earlier layers; each layer's first call joins them
            # (network workloads: only the network input and the loss gradient)
            for i, d in enumerate(L):
                if not NET or i == 0:
                    dc.dc_tensor_import(d["plan"], dc.DC_X, d["host"]["x"], d["xb"],
                                        IMPORT_SRC | dc.DC_IMPORT_ASYNC, sp)
                if not NET or i == len(L) - 1:
                    dc.dc_tensor_import(d["plan"], dc.DC_DY, d["host"]["dy"], d["dyb"],
                                        IMPORT_SRC | dc.DC_IMPORT_ASYNC, sp)
                d["w"].copy_(d["host"]["w"], non_blocking=True)
        for _, _, f in step_ops():
            f()
        dc.dc_comm_sync(comm, sp)
        if e2e:  # dW is final after the queued allreduces are joined
            for d in L:
                d["host"]["dw"].copy_(d["dw"], non_blocking=True)

    def barrier():
        if world > 1:
            dist.barrier()

    # CUDA graphs: the step's ~300 launches are recorded once and replayed, so
    # small layers are not bound by host launch cost (the P2P halo and BN
    # protocols keep their epochs on the device, so replays stay in step).
    use_graph = args.graph in ("on", "auto")

    def capture(fn):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream, capture_error_mode="thread_local"):
            fn()
        return g

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
        step(e2e=True)  # (sizes the import staging before any capture)
        torch.cuda.synchronize()
        if use_graph:
            g_step, g_e2e = capture(step), capture(lambda: step(e2e=True))
            g_ops = [(i, name, capture(lambda f=f: (f(), dc.dc_comm_sync(comm, sp)))) for i, name, f in step_ops()]
            run_step, run_e2e = g_step.replay, g_e2e.replay
            for _ in range(2):
                run_step()
            torch.cuda.synchronize()
        else:
            g_ops = None
            run_step, run_e2e = step, lambda: step(e2e=True)
        # ---- timed region: exactly K steps ----
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        clocks = ClockSampler(local)
        clocks.start()
        barrier()
        torch.cuda.synchronize()
        launches0 = dc.dc_kernel_launches()
        start.record(stream)
        for k in range(args.steps):
            run_step()
        stop.record(stream)
        torch.cuda.synchronize()
        launches = dc.dc_kernel_launches() - launches0
        barrier()
        clk = clocks.stop()
        ms = start.elapsed_time(stop)
        if use_graph:  # the replays launch the recorded kernels without calling the library
            launches0 = dc.dc_kernel_launches()
            step()
            torch.cuda.synchronize()
            launches = (dc.dc_kernel_launches() - launches0) * args.steps
        # ---- end-to-end leg: same steps with H2D of inputs / D2H of dW ----
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for k in range(args.steps):
            run_e2e()
        e1.record(stream)
        torch.cuda.synchronize()
        ms_e2e = e0.elapsed_time(e1)
        # ---- per-op device times: an instrumented pass, events between ops ----
        barrier()
        ops_list = g_ops if g_ops else step_ops()
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(len(ops_list) + 1)] for _ in range(args.steps)]
        for k in range(args.steps):
            ev[k][0].record(stream)
            for j, (i, name, f) in enumerate(ops_list):
                if g_ops:
                    f.replay()
                else:
                    f()
                    dc.dc_comm_sync(comm, sp)
                ev[k][j + 1].record(stream)
        torch.cuda.synchronize()

    t = torch.tensor([ms, ms_e2e], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, ms_e2e = float(t[0]), float(t[1])
    flops_step = sum(3 * layer_flops(d["l"]) for d in L)
    value = flops_step * args.steps / (ms / 1e3) / 1e12
    value_e2e = flops_step * args.steps / (ms_e2e / 1e3) / 1e12
    # the bytes step(e2e=True) copies: every layer's x, dy and w, or for a
    # network only the input x of the first layer and the loss gradient dy of
    # the last (the activations flow through the layers on the device)
    def nbytes(t):
        return t.numel() * t.element_size()
    h2d = sum(nbytes(d["host"]["w"]) + (nbytes(d["host"]["x"]) if not NET or i == 0 else 0) +
              (nbytes(d["host"]["dy"]) if not NET or i == len(L) - 1 else 0) for i, d in enumerate(L))
    d2h = sum(d["host"]["dw"].numel() * 4 for d in L)

    # ---- per-op device times on the launching stream, from the timed steps ----
    # median over the instrumented steps (one op hit by a stray clock dip must
    # not become the reported roofline kernel), indexed by (layer, op name)
    op_t = [dict() for _ in L]
    for j, (i, name, _) in enumerate(ops_list):
        op_t[i][name] = statistics.median(ev[k][j].elapsed_time(ev[k][j + 1]) for k in range(args.steps))
    per = []
    for i, d in enumerate(L):
        t = op_t[i]
        bwd = t.get("bwd", t.get("bpw", 0.0) + t.get("bpx", 0.0))
        d["bn_ms"] = t.get("bn", 0.0)
        per.append((d, t["fwd"], bwd, t))
    peaks, peak_src = load_peaks()
    # dominant kernel: conv_v2_kernel (the implicit-GEMM forward / backward-data
    # kernel, the largest share of the step in profiles/r1_launches_*.txt),
    # reported on the layer whose forward takes longest -- at one GPU that op
    # is exactly one conv_v2 launch (no split-K on the large layers).
    op_ms, d = max(((f_ms, d) for d, f_ms, b_ms, t in per), key=lambda c: c[0])
    op = "fp"
    loc = d["l"]
    # algorithmic work of THIS rank's shard (blocked split: global / world)
    fl = layer_flops(loc) / world
    by = layer_bytes(loc, op, 4 if fp32 else 2) / world
    tensor_peak, tensor_src = peaks["bf16_tflops"], "bf16 dense, measured burst (MEASURED_PEAKS.json)"
    if fp32:
        # 3xTF32: three tf32 tensor-core products per algorithmic multiply-add,
        # so the peak for algorithmic FLOPs is the measured dense tf32 rate / 3
        try:
            tf = json.load(open(os.path.join(ROOT, "profiles", "r2_tf32_peak.json")))["tf32_tflops"]
            tsrc = "measured burst, cuBLAS tf32 8192^3 (profiles/r2_tf32_peak.json)"
        except (OSError, ValueError, KeyError):
            tf, tsrc = peaks["bf16_tflops"] * 0.5, "bf16 measured x 0.5 (nominal tf32/bf16 ratio)"
        tensor_peak, tensor_src = tf / 3.0, f"tf32 dense {tf:.1f} TFLOP/s {tsrc}, / 3 products (3xTF32)"
    ridge = tensor_peak * 1e12 / (peaks["hbm_gbs"] * 1e9)
    if fl / by >= ridge:
        roof = {"bound": "tensor", "achieved": fl / (op_ms / 1e3) / 1e12, "peak": tensor_peak,
                "unit": "TFLOP/s"}
    else:
        roof = {"bound": "hbm", "achieved": by / (op_ms / 1e3) / 1e9, "peak": peaks["hbm_gbs"], "unit": "GB/s"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    # DRAM bytes per launch of this kernel on this shape from the committed
    # `ncu --set full` capture (profiles/r1_traffic.json), when there is one
    roof["traffic"] = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "r1_traffic.json")))
        key = f"conv_v2_kernel fwd {list(loc[1:])}"
        if world == 1 and key in tr:
            roof["traffic"] = tr[key]["dram_bytes"]
            roof["traffic_algorithmic"] = by
    except (OSError, ValueError, KeyError):
        pass
    roof["kernel"] = (f"conv_v2_kernel{'<tf32>' if fp32 else ''} ({loc[0]} forward"
                      f"{'' if world == 1 else ' incl. halo exchange'})")
    roof["avg_launch_ms"] = op_ms
    roof["peak_source"] = tensor_src if roof["bound"] == "tensor" else peak_src + " HBM copy (MEASURED_PEAKS.json)"

    out = None
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            import oracle
            oracle.build()
            f, s, desc = oracle_sample(layers, budget_s=15.0)
            cpu = {"value": f / s / 1e12, "unit": "TFLOP/s", "cores": oracle.num_threads(), "kind": "oracle",
                   "sample": desc}
        out = {
            **({"DIAGNOSTIC_ablated": sorted(ablate)} if ablate else {}),
            "metric": "conv fwd+bwd TFLOP/s", "value": value, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "fp32 (3xTF32: tf32 x3 products, fp32 accumulate)" if fp32 else "bf16",
            "data": "synthetic (seeded counter-based generator, " + (
                "fp32-exact 24-bit values)" if fp32 else "bf16-exact values)"),
            "config": {"workload": args.workload, "global_batch": layers[0][1],
                       "layers": [{"name": d["l"][0], "shape_NCHW_F_K_S_P": list(d["l"][1:]),
                                   "decomp": list(d["decomp"]), "model_pred_ms": d["pred"] * 1e3,
                                   "fwd_ms": f_ms, "bn_stats_ms": d["bn_ms"], "bwd_ms": b_ms,
                                   **({"bwd_filter_ms": t["bpw"], "bwd_data_ms": t["bpx"]} if "bpw" in t else {}),
                                   **({"bn_apply_relu_ms": t["act"]} if "act" in t else {}),
                                   **({"bn_relu_bwd_ms": t["bnb"]} if "bnb" in t else {}),
                                   **({"shuffle_fwd_ms": t["shuf"]} if "shuf" in t else {}),
                                   **({"shuffle_bwd_ms": t["shufb"]} if "shufb" in t else {}),
                                   "fwd_tflops": layer_flops(d["l"]) / (f_ms / 1e3) / 1e12,
                                   "bwd_tflops": 2 * layer_flops(d["l"]) / (b_ms / 1e3) / 1e12}
                                  for d, f_ms, b_ms, t in per],
                       "network": ("end to end: conv -> spatial BN -> BN apply + ReLU into the next layer's "
                                   "margined input; backward through BN / ReLU (group sums) into the previous "
                                   "layer's margined dy; " + (
                                       f"one grid per layer (model strategy), {n_shuffles} redistributions "
                                       "each way" if strategy else "one grid for all layers")) if NET else
                                  "conv stack: every layer on its own resident inputs",
                       **({"strategy": strategy} if strategy else {}),
                       "parallelism": {"auto": "per-layer model-chosen (pN,pH,pW)",
                                       "spatial": "pure spatial, per-layer model-chosen (1,pH,pW)",
                                       "strategy": "model strategy: per-layer grids + redistribution"}.get(
                                           args.decomp, args.decomp),
                       "halo": args.halo + ("+no-overlap" if args.no_overlap else ""), "l2": "working set per step > L2 (126 MB); no explicit flush",
                       "perf_model_table": os.path.relpath(table, ROOT) if table else "roofline estimate",
                       "perf_model_comm": MODEL_COMM,
                       "cuda_graph": use_graph, "dw_allreduce": "sync" if args.ar_sync else "async (joined at step end)",
                       "per_layer_times": "instrumented pass after the timed region (events between ops; median over its steps)",
                       "flops_per_step": flops_step},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": value_e2e, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        print(json.dumps(out), file=JSON_OUT, flush=True)
    if args.cost_table and rank == 0:
        with open(args.cost_table, "w") as f:
            f.write("op,n,c,h,w,f,k,s,pad,seconds\n")
            for d, f_ms, b_ms, t in per:
                _, N, C, H, W, F, K, S, P = d["l"]
                xd = d["xd"]
                for op, tt in (("fp", f_ms), ("bpw", t.get("bpw")), ("bpx", t.get("bpx"))):
                    if tt is not None:
                        f.write(f"{op},{xd['n']},{C},{xd['h']},{xd['w']},{F},{K},{S},{P},{tt / 1e3}\n")
    # teardown watchdog: a teardown stuck for 120 s prints every thread's stack
    # to stderr and exits (the result line is already out)
    faulthandler.dump_traceback_later(120, exit=True)
    # graphs hold NCCL persistent resources: release every reference to them
    # (the per-op list included) before the communicator
    del run_step, run_e2e
    g_step = g_e2e = g_ops = ops = f = ops_list = None
    import gc
    gc.collect()
    torch.cuda.synchronize()
    for d in L:
        for k in ("r_fwd", "r_bwd"):
            if k in d:
                dc.dc_redist_destroy(d[k])
    for d in L:
        dc.dc_plan_destroy(d["plan"])
    if world > 1:
        # every rank is done and its line is out: leave without the NCCL
        # teardown, which was measured to block in the multi-rank bench
        # (communicators whose collectives were captured into CUDA graphs);
        # the driver owns the processes, and exit releases the devices
        torch.cuda.synchronize()
        dist.barrier()
        sys.stdout.flush()
        sys.stderr.flush()
        os._exit(0)
    dc.dc_comm_destroy(comm)
    faulthandler.cancel_dump_traceback_later()


if __name__ == "__main__":
    main()
