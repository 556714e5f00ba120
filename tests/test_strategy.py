"""NEXT-3: the Shuffle(D_i, D_j) cost of a redistribution
 and the parallel execution strategy search
 -- the product (perfmodel.cpp) against the oracle
(oracle/perfmodel.py: element-by-element ownership counting, exhaustive
enumeration of strategies), and the oracle against hand-priced values."""
import os
import tempfile

import pytest

import oracle
from oracle import partition as part
from oracle import perfmodel as pm

A, B = 2e-6, 1.0 / 500e9


@pytest.fixture(scope="module")
def dc():
    from paper_1903_06681_b200 import build
    build.build()
    import paper_1903_06681_b200 as dc
    return dc


def test_shuffle_oracle_hand_priced():
    """(4,1,1) -> (1,4,1) of a 4 x 2 x 8 x 3 activation: each rank keeps the
    rows of its own sample it owns under both and sends 1 sample x 2 rows x 3
    cols x 2 channels = 12 words to each of its 3 peers: 3 SR(12 words of 2 B)."""
    assert pm.shuffle_cost(4, 2, 8, 3, (4, 1, 1), (4, 1, 1), A, B) == 0.0
    want = 3 * (A + 12 * 2 * B)
    assert abs(pm.shuffle_cost(4, 2, 8, 3, (4, 1, 1), (1, 4, 1), A, B) - want) < 1e-18
    w = pm.shuffle_words(4, 2, 8, 3, (4, 1, 1), (1, 4, 1))
    assert len(w) == 12 and set(w.values()) == {12}
    # H split -> W split of 1 x 1 x 4 x 4 (2 ranks): each sends a 2 x 2 quarter
    w = pm.shuffle_words(1, 1, 4, 4, (1, 2, 1), (1, 1, 2))
    assert w == {(0, 1): 4, (1, 0): 4}


@pytest.mark.parametrize("shape,pair", [
    ((8, 16, 32, 24), ((8, 1, 1), (1, 4, 2))),
    ((8, 16, 32, 24), ((2, 2, 2), (1, 8, 1))),
    ((4, 64, 17, 13), ((1, 2, 2), (2, 1, 2))),
    ((3, 8, 20, 20), ((1, 3, 1), (1, 1, 3))),
    ((6, 8, 12, 10), ((2, 3, 1), (3, 1, 2))),
])
def test_shuffle_cost_matches_oracle(dc, shape, pair):
    dc.dc_model_set_comm(A, B)
    N, Ch, H, W = shape
    for src, dst in (pair, pair[::-1]):
        got = dc.dc_model_shuffle_cost(N, Ch, H, W, src, dst)
        want = pm.shuffle_cost(N, Ch, H, W, src, dst, A, B)
        assert abs(got - want) <= 1e-12 * max(want, 1e-9), (src, dst, got, want)


def _load_table(dc, layers, worlds):
    def cost(op, n, c, h, w, f):
        return 1e-6 * (1 + {"fp": 1, "bpx": 2, "bpw": 3}[op]) * (n * c * h * w * f) ** 0.5 / 50
    rows = ["op,n,c,h,w,f,k,s,pad,seconds"]
    for l in layers:
        for P_tot in worlds:
            for g in pm.candidates(P_tot):
                if not pm.valid(l, g):
                    continue
                n = part.blocked(l["N"], g[0], 0)[1]
                h = part.blocked(l["H"], g[1], 0)[1]
                w = part.blocked(l["W"], g[2], 0)[1]
                for op in ("fp", "bpx", "bpw"):
                    rows.append(f"{op},{n},{l['C']},{h},{w},{l['F']},{l['K']},{l['S']},{l['P']},"
                                f"{cost(op, n, l['C'], h, w, l['F'])!r}")
    with tempfile.NamedTemporaryFile("w", suffix=".csv", delete=False) as f:
        f.write("\n".join(rows) + "\n")
    dc.dc_model_load_table(f.name)
    os.unlink(f.name)
    return cost


def _chain(specs):
    """[(C, H, F, K, S, P)] at N -> oracle layer dicts, parents, C-ABI tuples."""
    layers, parents, abi = [], [], []
    for i, (N, C, H, F, K, S, P, par) in enumerate(specs):
        layers.append(dict(N=N, C=C, H=H, W=H, F=F, K=K, S=S, P=P))
        parents.append(par)
        abi.append((N, C, H, H, F, K, S, P, par[0], par[1] if len(par) > 1 else -1))
    return layers, parents, abi


LINE = [(4, 16, 16, 32, 3, 1, 1, [-1]), (4, 32, 16, 64, 3, 2, 1, [0]), (4, 64, 8, 64, 3, 1, 1, [1]),
        (4, 64, 8, 128, 1, 1, 0, [2])]
BRANCHED = [(2, 16, 16, 32, 3, 1, 1, [-1]),            # 0
            (2, 32, 16, 32, 3, 1, 1, [0]),             # 1: main path
            (2, 32, 16, 64, 1, 1, 0, [1]),             # 2
            (2, 32, 16, 64, 1, 1, 0, [0]),             # 3: shortcut projection
            (2, 64, 16, 32, 3, 1, 1, [2, 3])]          # 4: reads the residual join


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("overlap", [True, False])
def test_line_strategy_is_the_exhaustive_optimum(dc, world, overlap):
    """A line network: the shortest path's total equals the
    minimum over every assignment of valid grids, and the grids it returns
    price to that total under the oracle's definitions."""
    layers, parents, abi = _chain(LINE)
    cost = _load_table(dc, layers, [world])
    dc.dc_model_set_comm(A, B)
    dc.dc_model_set_overlap(overlap)
    try:
        grids, total = dc.dc_model_strategy(abi, world)
        best_grids, best = pm.strategy_exhaustive(layers, parents, world, cost, A, B, overlap=overlap)
        assert abs(total - best) <= 1e-12 * best, (total, best, grids, best_grids)
        again = pm.strategy_total(layers, parents, grids, cost, A, B, overlap=overlap)
        assert abs(again - total) <= 1e-12 * total
        # pure spatial restriction
        g1, t1 = dc.dc_model_strategy(abi, world, fix_pn=1)
        assert all(g[0] == 1 for g in g1) and t1 >= total - 1e-15
    finally:
        dc.dc_model_set_overlap(True)


@pytest.mark.parametrize("world", [2, 4])
def test_branched_strategy(dc, world):
    """A network with a residual join: the longest-path
    heuristic returns a valid assignment whose reported total is the oracle's
    price of it, no better than the exhaustive optimum."""
    layers, parents, abi = _chain(BRANCHED)
    cost = _load_table(dc, layers, [world])
    dc.dc_model_set_comm(A, B)
    grids, total = dc.dc_model_strategy(abi, world)
    assert all(pm.valid(l, g) for l, g in zip(layers, grids))
    assert abs(pm.strategy_total(layers, parents, grids, cost, A, B) - total) <= 1e-12 * total
    _, best = pm.strategy_exhaustive(layers, parents, world, cost, A, B)
    assert total >= best - 1e-15


def test_strategy_errors(dc):
    with pytest.raises(dc.DCError):   # child does not read the parent's output shape
        dc.dc_model_strategy([(1, 8, 16, 16, 8, 3, 1, 1, -1), (1, 16, 16, 16, 8, 3, 1, 1, 0)], 2)
    with pytest.raises(dc.DCError):   # parent after the child
        dc.dc_model_strategy([(1, 8, 16, 16, 8, 3, 1, 1, 1), (1, 8, 16, 16, 8, 3, 1, 1, -1)], 2)
