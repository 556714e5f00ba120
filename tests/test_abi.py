"""The C-ABI library loads on a CPU-only box and exports every symbol that
include/dconv.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def dc():
    from paper_1903_06681_b200 import build
    build.build()
    import paper_1903_06681_b200 as dc
    return dc


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "dconv.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dc_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported(dc):
    L = ctypes.CDLL(dc.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), f"{s} declared in include/dconv.h but not exported"
    assert sorted(dc.EXPORTS) == syms


def test_errors_are_status_codes_not_exceptions(dc):
    with pytest.raises(dc.DCError) as e:
        dc.dc_plan_create_virtual(1, 2, 16, 16, 4, 4, 1, 1, (1, 1, 1), 0)   # even K
    assert e.value.status == dc.DC_ERR_SHAPE
    with pytest.raises(dc.DCError) as e:
        dc.dc_plan_create_virtual(1, 2, 16, 16, 4, 3, 3, 1, (1, 1, 1), 0)   # stride 3
    assert e.value.status == dc.DC_ERR_UNSUPPORTED
    with pytest.raises(dc.DCError) as e:
        dc.dc_plan_create_virtual(1, 2, 16, 16, 4, 3, 1, 2, (1, 1, 1), 0)   # P > K/2
    assert e.value.status == dc.DC_ERR_SHAPE
    with pytest.raises(dc.DCError) as e:
        dc.dc_plan_create_virtual(1, 2, 16, 16, 4, 3, 1, 1, (2, 1, 1), 0)   # pN > N
    assert e.value.status == dc.DC_ERR_PARTITION
    with pytest.raises(dc.DCError) as e:
        dc.dc_plan_create_virtual(1, 1, 8, 8, 1, 7, 1, 3, (1, 4, 1), 0)
    assert e.value.status == dc.DC_ERR_PARTITION
    with pytest.raises(dc.DCError) as e:
        dc.dc_plan_create_virtual(1, 2, 16, 16, 4, 3, 1, 1, (1, 1, 1), 0, dtype=7)     # unknown dtype
    assert e.value.status == dc.DC_ERR_ARG
    # the thread-local message of the last failing call names the cause
    assert "dtype" in str(e.value), str(e.value)
    assert dc.lib().dc_last_error().decode() in str(e.value)


def test_fp32_plan_layouts(dc):
    """DC_FP32_3XTF32 plans: channels padded to 8 (C <= 8) or 32, margined
    x / dy hold [hi | lo] fp32 halves, y / dx plain fp32, w fp32, dW unpadded."""
    p = dc.dc_plan_create_virtual(2, 18, 20, 20, 12, 3, 1, 1, (1, 2, 1), 0, dtype=dc.DC_FP32_3XTF32)
    try:
        x, y = dc.dc_plan_query(p, dc.DC_X), dc.dc_plan_query(p, dc.DC_Y)
        dy, w, dw = dc.dc_plan_query(p, dc.DC_DY), dc.dc_plan_query(p, dc.DC_W), dc.dc_plan_query(p, dc.DC_DW)
        assert (x["c"], x["c_pad"], x["halo_s"]) == (18, 2 * 32, 1)
        assert x["bytes"] == 2 * x["hb"] * x["wb"] * 64 * 4
        assert (y["c_pad"], y["bytes"]) == (32, 2 * 10 * 20 * 32 * 4)
        assert (dy["c_pad"], w["c_pad"], w["bytes"]) == (64, 32, 12 * 9 * 32 * 4)
        assert (dw["c_pad"], dw["bytes"]) == (18, 12 * 9 * 18 * 4)
        p2 = dc.dc_plan_create_virtual(1, 3, 8, 8, 4, 3, 1, 1, (1, 1, 1), 0, dtype=dc.DC_FP32_3XTF32)
        assert dc.dc_plan_query(p2, dc.DC_X)["c_pad"] == 2 * 8 and dc.dc_plan_query(p2, dc.DC_Y)["c_pad"] == 8
        dc.dc_plan_destroy(p2)
    finally:
        dc.dc_plan_destroy(p)


def test_c1_shard_descriptors(dc):
    """Config C1 (BASELINE.json configs[0]): N=1 C=2 H=W=16 F=4 K=3 P=1, 2-way H."""
    for rank in range(2):
        p = dc.dc_plan_create_virtual(1, 2, 16, 16, 4, 3, 1, 1, (1, 2, 1), rank)
        x = dc.dc_plan_query(p, dc.DC_X)
        assert (x["h0"], x["h"], x["w"], x["c"], x["c_pad"]) == (8 * rank, 8, 16, 2, 16)
        assert (x["halo_n"], x["halo_s"]) == ((0, 1) if rank == 0 else (1, 0))
        assert x["bytes"] == 1 * 9 * 16 * 16 * 2
        y = dc.dc_plan_query(p, dc.DC_Y)
        assert (y["h0"], y["h"], y["c_pad"]) == (8 * rank, 8, 16)
        assert dc.dc_plan_decomp(p)[0] == (1, 2, 1)
        dc.dc_plan_destroy(p)
