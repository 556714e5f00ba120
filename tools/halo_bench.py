"""Halo-exchange microbenchmark over NVLink (direct P2P stores vs the NCCL
send/recv baseline), one process per GPU:

  torchrun --nproc-per-node 2 tools/halo_bench.py

For each layer (shapes of the mesh2k_n8 stack plus larger slabs) and each
transport, times 50 back-to-back dc_halo_exchange calls of x on the layer's
pure H split, captured in one CUDA graph and replayed, with CUDA events
(after warm-up and a barrier; max over ranks)
and reports the bytes each rank sends per exchange, the time per exchange and
the achieved send bandwidth per GPU (GB/s, NVLink 5: 900 GB/s per direction).
Prints one JSON line per case on rank 0."""
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1903_06681_b200 as dc  # noqa: E402

CASES = [  # (name, N, C, H, W, F, K, S, P)
    ("conv1_2", 8, 64, 1024, 1024, 64, 3, 1, 1),
    ("conv2_2", 8, 128, 512, 512, 128, 3, 1, 1),
    ("conv3_2", 8, 256, 256, 256, 256, 3, 1, 1),
    ("conv4_2", 8, 512, 128, 128, 512, 3, 1, 1),
    ("conv6_2", 8, 512, 32, 32, 512, 3, 1, 1),
    ("slab_k7_c256", 8, 256, 512, 1024, 256, 7, 1, 3),
]


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    uid = [dc.dc_comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = dc.dc_comm_create(rank, world, uid[0], local)
    s = torch.cuda.Stream()
    for name, N, C, H, W, F, K, S, P in CASES:
        plan = dc.dc_plan_create(N, C, H, W, F, K, S, P, (1, world, 1), dc.DC_BF16, comm)
        xd = dc.dc_plan_query(plan, dc.DC_X)
        buf = dc.dc_buffer_alloc(plan, dc.DC_X)
        sent = sum(m["rows"] * m["cols"] for m in dc.dc_plan_halo_msgs(plan, dc.DC_X) if m["is_send"])
        sent_bytes = sent * xd["n"] * xd["c_pad"] * 2
        for label, flags in (("p2p", 0), ("nccl", dc.DC_HALO_NCCL)):
            reps = 50
            with torch.cuda.stream(s):
                for _ in range(5):
                    dc.dc_halo_exchange(plan, dc.DC_X, buf, flags, s)
                torch.cuda.synchronize()
                # the 50 exchanges replayed from one CUDA graph: device time,
                # not the host's per-call launch cost
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    for _ in range(reps):
                        dc.dc_halo_exchange(plan, dc.DC_X, buf, flags, s)
                torch.cuda.synchronize()
                dist.barrier()
                g.replay()
                torch.cuda.synchronize()
                dist.barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                g.replay()
                e1.record(s)
                torch.cuda.synchronize()
                del g
            t = torch.tensor([e0.elapsed_time(e1) / reps], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            b = torch.tensor([float(sent_bytes)], dtype=torch.float64, device="cuda")
            dist.all_reduce(b, op=dist.ReduceOp.MAX)
            if rank == 0:
                us = float(t[0]) * 1e3
                print(json.dumps({"case": name, "transport": label, "world": world, "grid": [1, world, 1],
                                  "bytes_sent_per_rank": int(b[0]), "us_per_exchange": round(us, 2),
                                  "send_GBps_per_gpu": round(float(b[0]) / (us * 1e-6) / 1e9, 1)}), flush=True)
        dc.dc_plan_destroy(plan)
    dc.dc_comm_destroy(comm)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
