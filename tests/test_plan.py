"""Host-side plan (L1) and performance model (L4) of libdconv checked against
the oracle: brute-force halo dependence sets, blocked
splits, send/recv duality, validity, and the paper's cost formulas."""
import itertools
import os
import tempfile

import pytest

from oracle import out_extent
from oracle import partition as part
from oracle import perfmodel as pm


@pytest.fixture(scope="module")
def dc():
    from paper_1903_06681_b200 import build
    build.build()
    import paper_1903_06681_b200 as dc
    return dc


CASES = []
for K, S in itertools.product([1, 3, 5, 7], [1, 2]):
    for P in sorted({0, K // 2}):
        for H, W in [(17, 13), (24, 24), (9, 30)]:
            for grid in [(1, 1, 1), (1, 2, 1), (1, 1, 2), (1, 2, 2), (2, 3, 1), (1, 4, 4), (1, 3, 2)]:
                CASES.append((K, S, P, H, W, grid))


def _grid_ok(layer, grid):
    return pm.valid(layer, grid)


@pytest.mark.parametrize("K,S,P,H,W,grid", CASES)
def test_halo_matches_bruteforce(dc, K, S, P, H, W, grid):
    N = 2
    layer = dict(N=N, C=3, H=H, W=W, F=5, K=K, S=S, P=P)
    ok = _grid_ok(layer, grid)
    ranks = grid[0] * grid[1] * grid[2]
    if not ok:
        with pytest.raises(dc.DCError) as e:
            dc.dc_plan_create_virtual(N, 3, H, W, 5, K, S, P, grid, 0)
        assert e.value.status == dc.DC_ERR_PARTITION
        return
    Ho, Wo = out_extent(H, K, S, P), out_extent(W, K, S, P)
    msgs = {}
    for r in range(ranks):
        p = dc.dc_plan_create_virtual(N, 3, H, W, 5, K, S, P, grid, r)
        iN, iH, iW = part.rank_coords(r, grid)
        x = dc.dc_plan_query(p, dc.DC_X)
        dy = dc.dc_plan_query(p, dc.DC_DY)
        # blocked splits
        assert (x["n0"], x["n"]) == (lambda a: (a[0], a[1] - a[0]))(part.blocked(N, grid[0], iN))
        for dim, ext, idx, parts, key0, key in ((0, H, iH, grid[1], "h0", "h"), (1, W, iW, grid[2], "w0", "w")):
            q, rr = part.blocked(ext, parts, idx)
            assert (x[key0], x[key]) == (q, rr - q)
            oq, orr = part.blocked(out_extent(ext, K, S, P), parts, idx)
            assert (dy[key0], dy[key]) == (oq, orr - oq)
            # x halo == brute-force dependence set minus owned rows, contiguous
            lo, hi = part.halo_rows(parts, idx, ext, K, S, P, "x")
            hl, hh = (x["halo_n"], x["halo_s"]) if dim == 0 else (x["halo_w"], x["halo_e"])
            assert sorted(lo) == list(range(q - hl, q)), (dim, idx)
            assert sorted(hi) == list(range(rr, rr + hh)), (dim, idx)
            lo, hi = part.halo_rows(parts, idx, ext, K, S, P, "dy")
            hl, hh = (dy["halo_n"], dy["halo_s"]) if dim == 0 else (dy["halo_w"], dy["halo_e"])
            assert sorted(lo) == list(range(oq - hl, oq)), ("dy", dim, idx)
            assert sorted(hi) == list(range(orr, orr + hh)), ("dy", dim, idx)
        if K == 1 and S == 1:  # PAPER.md:139 (stated for S=1; with S=2 blocked in/out splits can misalign)
            assert x["hb"] == x["h"] and x["wb"] == x["w"]
        for t in (dc.DC_X, dc.DC_DY):
            msgs[(r, t)] = dc.dc_plan_halo_msgs(p, t)
        dc.dc_plan_destroy(p)
    # send/recv duality: p's recv from q == q's send to p
    for t in (dc.DC_X, dc.DC_DY):
        for r in range(ranks):
            for m in msgs[(r, t)]:
                if m["is_send"]:
                    continue
                dual = [s for s in msgs[(m["peer"], t)] if s["is_send"] and s["peer"] == r]
                assert len(dual) == 1
                for k in ("row0", "rows", "col0", "cols"):
                    assert dual[0][k] == m[k]
        # total received = the halo region of the buffer (8 blocks)
        for r in range(ranks):
            p = dc.dc_plan_create_virtual(N, 3, H, W, 5, K, S, P, grid, r)
            d = dc.dc_plan_query(p, t)
            dc.dc_plan_destroy(p)
            recv = sum(m["rows"] * m["cols"] for m in msgs[(r, t)] if not m["is_send"])
            assert recv == d["hb"] * d["wb"] - d["h"] * d["w"]


def test_conv1_and_mesh_examples(dc):
    # ResNet-50 conv1 2-way: rank0 2 south rows, rank1 3 north rows
    p0 = dc.dc_plan_create_virtual(32, 3, 224, 224, 64, 7, 2, 3, (1, 2, 1), 0)
    p1 = dc.dc_plan_create_virtual(32, 3, 224, 224, 64, 7, 2, 3, (1, 2, 1), 1)
    assert dc.dc_plan_query(p0, dc.DC_X)["halo_s"] == 2
    assert dc.dc_plan_query(p1, dc.DC_X)["halo_n"] == 3
    # stride-2 3x3 P=1, 8-way on 2048 rows: rank 0 none, others one north row
    for r in range(8):
        p = dc.dc_plan_create_virtual(1, 18, 2048, 2048, 64, 3, 2, 1, (1, 8, 1), r)
        x = dc.dc_plan_query(p, dc.DC_X)
        assert (x["halo_n"], x["halo_s"]) == ((0, 0) if r == 0 else (1, 0))
        dc.dc_plan_destroy(p)


# ---------------- performance model vs the oracle's formulas ----------------

LAYERS = [dict(N=8, C=64, H=256, W=256, F=64, K=3, S=1, P=1),
          dict(N=32, C=3, H=224, W=224, F=64, K=7, S=2, P=3),
          dict(N=32, C=512, H=28, W=28, F=128, K=1, S=1, P=0),
          dict(N=1, C=18, H=2048, W=2048, F=64, K=3, S=1, P=1)]


def _table_cost(layer):
    """A synthetic empirical table with arbitrary values, used
    identically by the product (through the CSV) and the oracle."""
    def cost(op, n, c, h, w, f):
        return 1e-6 * (1 + {"fp": 1, "bpx": 2, "bpw": 3}[op]) * (n * c * h * w * f) ** 0.5 / 100
    return cost


@pytest.mark.parametrize("overlap,alpha_w", [(True, 0.0), (False, 0.0), (False, 4e-6)])
@pytest.mark.parametrize("layer", LAYERS)
def test_model_matches_oracle(dc, layer, overlap, alpha_w):
    alpha, beta = 3e-6, 1.0 / 600e9
    dc.dc_model_set_comm(alpha, beta)
    dc.dc_model_set_overlap(overlap)
    dc.dc_model_set_strided_latency(alpha_w)
    cost = _table_cost(layer)
    rows = ["op,n,c,h,w,f,k,s,pad,seconds"]
    for P_tot in (1, 2, 4, 8):
        for g in pm.candidates(P_tot):
            if not pm.valid(layer, g):
                continue
            n = part.blocked(layer["N"], g[0], 0)[1]
            h = part.blocked(layer["H"], g[1], 0)[1]
            w = part.blocked(layer["W"], g[2], 0)[1]
            for op in ("fp", "bpx", "bpw"):
                rows.append(f"{op},{n},{layer['C']},{h},{w},{layer['F']},{layer['K']},{layer['S']},{layer['P']},"
                            f"{cost(op, n, layer['C'], h, w, layer['F'])!r}")
    with tempfile.NamedTemporaryFile("w", suffix=".csv", delete=False) as f:
        f.write("\n".join(rows) + "\n")
    dc.dc_model_load_table(f.name)
    os.unlink(f.name)
    args = [layer[k] for k in ("N", "C", "H", "W", "F", "K", "S", "P")]
    for P_tot in (1, 2, 4, 8):
        for g in pm.candidates(P_tot):
            if not pm.valid(layer, g):
                with pytest.raises(dc.DCError):
                    dc.dc_model_layer_cost(*args, g)
                continue
            got = dc.dc_model_layer_cost(*args, g)
            want = pm.layer_cost(layer, g, cost, alpha, beta, overlap=overlap, alpha_w=alpha_w)["total"]
            assert abs(got - want) <= 1e-12 * max(1.0, want), (g, got, want)
        best, t = dc.dc_model_choose(*args, P_tot)
        ob, ot = pm.choose(layer, P_tot, cost, alpha, beta, overlap=overlap, alpha_w=alpha_w)
        assert best == ob and abs(t - ot) <= 1e-12 * max(1.0, ot)
        # pure spatial (p_N fixed to 1): the argmin of the oracle's costs over those grids,
        # first in the enumeration order on ties (larger p_H first, reading R17)
        spatial = [g for g in pm.candidates(P_tot) if g[0] == 1 and pm.valid(layer, g)]
        if spatial:
            costs = [pm.layer_cost(layer, g, cost, alpha, beta, overlap=overlap, alpha_w=alpha_w)["total"] for g in spatial]
            want = spatial[min(range(len(spatial)), key=lambda i: (costs[i], -spatial[i][1]))]
            got, ts = dc.dc_model_choose_fixed(*args, P_tot, (1, 0, 0))
            assert got == want and abs(ts - min(costs)) <= 1e-12 * max(1.0, ts), (got, want)
        else:
            with pytest.raises(dc.DCError):
                dc.dc_model_choose_fixed(*args, P_tot, (1, 0, 0))
    dc.dc_model_set_overlap(True)
    dc.dc_model_set_strided_latency(0.0)


@pytest.mark.gpu
def test_plan_create_partial_decomp(dc):
    """dc_plan_create with zero entries lets the model choose those (here on
    one rank: the only grid)."""
    for decomp in ((0, 0, 0), (1, 0, 0), (0, 1, 0), (1, 1, 0)):
        plan = dc.dc_plan_create(1, 18, 64, 64, 16, 3, 1, 1, decomp)
        assert dc.dc_plan_decomp(plan)[0] == (1, 1, 1)
        dc.dc_plan_destroy(plan)


def test_plan_create_partial_decomp_errors(dc):
    """Fixed entries that cannot cover the world, or negative ones, fail
    before any device work."""
    with pytest.raises(dc.DCError):
        dc.dc_plan_create(2, 18, 64, 64, 16, 3, 1, 1, (2, 0, 0))  # p_N = 2 on one rank
    with pytest.raises(dc.DCError):
        dc.dc_plan_create(1, 18, 64, 64, 16, 3, 1, 1, (-1, 0, 0))
