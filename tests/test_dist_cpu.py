"""World-size-2 (and 4) gloo tests on CPU of the N>1 host logic: each rank
plans its own shard (virtual plans, no GPU), the ranks exchange their halo
message lists over torch.distributed and check send/recv duality and halo
byte conservation against the paper's model terms, and
the max-over-ranks timing reduction bench.py uses."""
import os
import socket
import traceback

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


GRIDS = {2: [(1, 2, 1), (1, 1, 2), (2, 1, 1)], 4: [(1, 2, 2), (1, 4, 1), (2, 2, 1), (4, 1, 1)]}


def _worker(rank, world, port, q):
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import paper_1903_06681_b200 as dc
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        for grid in GRIDS[world]:
            for shape in [(4, 16, 64, 48, 32, 3, 1, 1), (4, 3, 224, 224, 64, 7, 2, 3), (4, 64, 56, 56, 64, 5, 1, 2)]:
                N, C, H, W, F, K, S, P = shape
                plan = dc.dc_plan_create_virtual(N, C, H, W, F, K, S, P, grid, rank)
                mine = {t: dc.dc_plan_halo_msgs(plan, t) for t in (dc.DC_X, dc.DC_DY)}
                desc = dc.dc_plan_query(plan, dc.DC_X)
                dc.dc_plan_destroy(plan)
                allm = [None] * world
                dist.all_gather_object(allm, (mine, desc))
                for t in (dc.DC_X, dc.DC_DY):
                    for m in mine[t]:
                        peer_msgs = allm[m["peer"]][0][t]
                        dual = [p for p in peer_msgs if p["peer"] == rank and p["is_send"] != m["is_send"]]
                        assert len(dual) == 1, (grid, shape, t, m)
                        assert all(dual[0][k] == m[k] for k in ("row0", "rows", "col0", "cols"))
                # the owned blocks tile the global tensor (coverage / disjointness)
                cells = sum(d["n"] * d["h"] * d["w"] for _, d in allm)
                assert cells == N * H * W
        # bench.py's device-time reduction: MAX over ranks
        t = torch.tensor([float(rank + 1), 10.0 * (world - rank)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        assert t.tolist() == [float(world), 10.0 * world]
        # allreduce of [rank] over 4 ranks -> [6]
        s = torch.tensor([float(rank)])
        dist.all_reduce(s)
        assert s.item() == world * (world - 1) / 2
        dist.destroy_process_group()
    except Exception:
        q.put(traceback.format_exc())
        raise


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_ranks(world):
    from paper_1903_06681_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=300)
    errs = []
    while not q.empty():
        errs.append(q.get())
    assert not errs and all(p.exitcode == 0 for p in ps), "\n".join(errs)
