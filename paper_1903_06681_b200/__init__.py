"""paper_1903_06681_b200 -- B200-native spatially / hybrid sample-spatial
partitioned convolution (Dryden et al., arXiv:1903.06681).

Thin ctypes binding of libdconv.so (include/dconv.h): the same entry points,
argument marshalling only. Every step of the hot path runs in the library's
sm_100a kernels and NCCL; nothing here computes. Importing fails loudly if
the shared library is missing (build it with
`python -m paper_1903_06681_b200.build`); there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdconv.so")

DC_OK, DC_ERR_ARG, DC_ERR_SHAPE, DC_ERR_PARTITION, DC_ERR_UNSUPPORTED, DC_ERR_CUDA, DC_ERR_COMM, DC_ERR_OOM = range(8)
STATUS_NAMES = ["DC_OK", "DC_ERR_ARG", "DC_ERR_SHAPE", "DC_ERR_PARTITION", "DC_ERR_UNSUPPORTED",
                "DC_ERR_CUDA", "DC_ERR_COMM", "DC_ERR_OOM"]
DC_BF16, DC_FP32_3XTF32 = 0, 1
DC_X, DC_Y, DC_DY, DC_DX, DC_W, DC_DW = range(6)
DC_EXCHANGE, DC_ALLREDUCE, DC_HALO_NCCL, DC_ALLREDUCE_ASYNC, DC_BN_STATS, DC_DETERMINISTIC, DC_DW_ATOMIC = (
    0x1, 0x2, 0x4, 0x8, 0x10, 0x20, 0x40)
DC_NO_OVERLAP = 0x80
DC_FORCE_OVERLAP = 0x100
DC_DEFAULT_FLAGS = DC_EXCHANGE | DC_ALLREDUCE
DC_BN_LOCAL, DC_BN_FROM_FWD = 0x1, 0x2
DC_IMPORT_ASYNC, DC_SRC_BF16 = 0x1, 0x2
DC_RELU = 0x4

# every symbol include/dconv.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "dc_comm_create", "dc_comm_create_local", "dc_comm_stream", "dc_comm_unique_id", "dc_comm_destroy", "dc_comm_sync",
    "dc_comm_set_bucket_bytes", "dc_plan_create",
    "dc_plan_create_virtual", "dc_plan_halo_msgs", "dc_plan_query", "dc_plan_decomp", "dc_plan_set_splitk_world",
    "dc_plan_destroy", "dc_buffer_alloc", "dc_tensor_import", "dc_halo_exchange", "dc_conv_fwd", "dc_conv_bwd_data",
    "dc_conv_bwd_filter", "dc_conv_bwd", "dc_bn_spatial_stats", "dc_bn_apply", "dc_bn_backward",
    "dc_kernel_launches",
    "dc_last_error", "dc_model_set_comm", "dc_model_set_overlap", "dc_model_set_strided_latency", "dc_model_load_table", "dc_model_layer_cost",
    "dc_model_choose", "dc_model_choose_fixed", "dc_model_shuffle_cost", "dc_model_strategy",
    "dc_redist_create", "dc_redist_bytes", "dc_redistribute", "dc_redist_destroy",
    "dc_cplan_create", "dc_cplan_create_virtual", "dc_cplan_query", "dc_cconv_fwd", "dc_cconv_bwd_data",
    "dc_cconv_bwd_filter", "dc_cplan_destroy",
    "dc_pool_create", "dc_pool_plans", "dc_pool_fwd", "dc_pool_bwd", "dc_pool_destroy",
]


class dc_decomp_t(ctypes.Structure):
    _fields_ = [("pn", ctypes.c_int32), ("ph", ctypes.c_int32), ("pw", ctypes.c_int32)]


class dc_layer_t(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int64), ("C", ctypes.c_int64), ("H", ctypes.c_int64), ("W", ctypes.c_int64),
                ("F", ctypes.c_int64), ("K", ctypes.c_int32), ("stride", ctypes.c_int32), ("pad", ctypes.c_int32),
                ("parent", ctypes.c_int32), ("parent2", ctypes.c_int32)]


class dc_shard_desc_t(ctypes.Structure):
    _fields_ = [("n0", ctypes.c_int64), ("h0", ctypes.c_int64), ("w0", ctypes.c_int64),
                ("n", ctypes.c_int64), ("h", ctypes.c_int64), ("w", ctypes.c_int64),
                ("c", ctypes.c_int64), ("c_pad", ctypes.c_int64),
                ("halo_n", ctypes.c_int32), ("halo_s", ctypes.c_int32),
                ("halo_w", ctypes.c_int32), ("halo_e", ctypes.c_int32),
                ("hb", ctypes.c_int64), ("wb", ctypes.c_int64),
                ("stride_n", ctypes.c_int64), ("stride_h", ctypes.c_int64),
                ("stride_w", ctypes.c_int64), ("bytes", ctypes.c_size_t)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class dc_halo_msg_t(ctypes.Structure):
    _fields_ = [("peer", ctypes.c_int32), ("is_send", ctypes.c_int32), ("row0", ctypes.c_int64),
                ("rows", ctypes.c_int64), ("col0", ctypes.c_int64), ("cols", ctypes.c_int64)]


class DCError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < 8 else status}: {msg}")
        self.status = status


_lib = None


def lib() -> ctypes.CDLL:
    """Load libdconv.so (raises if it was not built: no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run `python -m paper_1903_06681_b200.build`")
    L = ctypes.CDLL(LIB_PATH)
    i64, i32, vp, st = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_int
    P = ctypes.POINTER
    sig = {
        "dc_comm_create": [i32, i32, vp, i32, P(vp)],
        "dc_comm_unique_id": [vp],
        "dc_comm_create_local": [i32, i32, P(vp)],
        "dc_comm_stream": [vp, P(vp)],
        "dc_comm_destroy": [vp],
        "dc_plan_set_splitk_world": [vp, i32],
        "dc_comm_sync": [vp, vp],
        "dc_comm_set_bucket_bytes": [vp, ctypes.c_size_t],
        "dc_plan_create": [i64] * 5 + [i32, i32, i32, dc_decomp_t, i32, vp, P(vp)],
        "dc_plan_create_virtual": [i64] * 5 + [i32, i32, i32, dc_decomp_t, i32, i32, P(vp)],
        "dc_plan_halo_msgs": [vp, i32, P(dc_halo_msg_t), P(i32)],
        "dc_plan_query": [vp, i32, P(dc_shard_desc_t)],
        "dc_plan_decomp": [vp, P(dc_decomp_t), P(ctypes.c_double)],
        "dc_plan_destroy": [vp],
        "dc_buffer_alloc": [vp, i32, P(vp)],
        "dc_halo_exchange": [vp, i32, vp, ctypes.c_uint, vp],
        "dc_tensor_import": [vp, i32, vp, vp, ctypes.c_uint, vp],
        "dc_conv_fwd": [vp, vp, vp, vp, ctypes.c_uint, vp],
        "dc_conv_bwd_data": [vp, vp, vp, vp, ctypes.c_uint, vp],
        "dc_conv_bwd_filter": [vp, vp, vp, vp, ctypes.c_uint, vp],
        "dc_conv_bwd": [vp, vp, vp, vp, vp, vp, ctypes.c_uint, vp],
        "dc_bn_spatial_stats": [vp, vp, vp, vp, ctypes.c_uint, vp],
        "dc_bn_apply": [vp, vp, vp, vp, vp, vp, ctypes.c_double, vp, ctypes.c_uint, vp, vp, vp],
        "dc_bn_backward": [vp, vp, vp, vp, vp, vp, vp, ctypes.c_double, vp, ctypes.c_uint, vp, vp, vp, vp, vp],
        "dc_model_set_comm": [ctypes.c_double, ctypes.c_double],
        "dc_model_load_table": [ctypes.c_char_p],
        "dc_model_set_overlap": [i32],
        "dc_model_set_strided_latency": [ctypes.c_double],
        "dc_model_layer_cost": [i64] * 5 + [i32, i32, i32, dc_decomp_t, i32, P(ctypes.c_double)],
        "dc_model_choose": [i64] * 5 + [i32, i32, i32, i32, P(dc_decomp_t), P(ctypes.c_double)],
        "dc_model_choose_fixed": [i64] * 5 + [i32, i32, i32, i32, dc_decomp_t, P(dc_decomp_t), P(ctypes.c_double)],
        "dc_model_shuffle_cost": [i64] * 4 + [dc_decomp_t, dc_decomp_t, P(ctypes.c_double)],
        "dc_model_strategy": [P(dc_layer_t), i32, i32, i32, P(dc_decomp_t), P(ctypes.c_double)],
        "dc_redist_create": [vp, i32, vp, i32, P(vp)],
        "dc_redist_bytes": [vp, P(i64), P(i64)],
        "dc_redistribute": [vp, vp, vp, ctypes.c_uint, vp],
        "dc_redist_destroy": [vp],
        "dc_cplan_create": [i64] * 5 + [i32, i32, i32, i32, i32, i32, vp, P(vp)],
        "dc_cplan_create_virtual": [i64] * 5 + [i32, i32, i32, i32, i32, i32, P(vp)],
        "dc_cplan_query": [vp, i32, P(dc_shard_desc_t), P(i64)],
        "dc_cconv_fwd": [vp, vp, vp, vp, ctypes.c_uint, vp],
        "dc_cconv_bwd_data": [vp, vp, vp, vp, ctypes.c_uint, vp],
        "dc_cconv_bwd_filter": [vp, vp, vp, vp, ctypes.c_uint, vp],
        "dc_cplan_destroy": [vp],
        "dc_pool_create": [i64] * 4 + [i32, i32, i32, dc_decomp_t, i32, vp, P(vp)],
        "dc_pool_plans": [vp, P(vp), P(vp)],
        "dc_pool_fwd": [vp, vp, vp, ctypes.c_uint, vp],
        "dc_pool_bwd": [vp, vp, vp, vp, ctypes.c_uint, vp],
        "dc_pool_destroy": [vp],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = st
    L.dc_last_error.restype = ctypes.c_char_p
    L.dc_last_error.argtypes = []
    L.dc_kernel_launches.restype = ctypes.c_uint64
    L.dc_kernel_launches.argtypes = []
    _lib = L
    return L


def _check(status: int):
    if status != DC_OK:
        raise DCError(status, lib().dc_last_error().decode(errors="replace"))


def _ptr(t) -> int | None:
    """Device/host pointer of a torch tensor (or an int address)."""
    if t is None:
        return None
    return t if isinstance(t, int) else t.data_ptr()


def _stream(s) -> int | None:
    if s is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return s if isinstance(s, int) else s.cuda_stream


# ---------------- same names as the C ABI ----------------

def dc_comm_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().dc_comm_unique_id(buf))
    return buf.raw


def dc_comm_create(rank: int, world: int, uid: bytes | None, device: int) -> int:
    out = ctypes.c_void_p()
    ub = ctypes.create_string_buffer(uid, 128) if uid is not None else None
    _check(lib().dc_comm_create(rank, world, ub, device, ctypes.byref(out)))
    return out.value


def dc_comm_create_local(world: int, device: int = 0) -> list[int]:
    """Loopback group: `world` virtual ranks of this process on one device."""
    arr = (ctypes.c_void_p * world)()
    _check(lib().dc_comm_create_local(world, device, arr))
    return [arr[i] for i in range(world)]


def dc_comm_stream(comm: int) -> int:
    """The compute stream (cudaStream_t) of a loopback rank."""
    out = ctypes.c_void_p()
    _check(lib().dc_comm_stream(comm, ctypes.byref(out)))
    return out.value


def dc_comm_destroy(comm: int):
    _check(lib().dc_comm_destroy(comm))


def dc_comm_sync(comm: int, stream=None):
    """Make `stream` wait for the dW allreduces queued with DC_ALLREDUCE_ASYNC."""
    _check(lib().dc_comm_sync(comm, _stream(stream)))


def dc_comm_set_bucket_bytes(comm: int, nbytes: int):
    """Bucket the DC_ALLREDUCE_ASYNC dW allreduces up to nbytes (0: none)."""
    _check(lib().dc_comm_set_bucket_bytes(comm, nbytes))


def dc_plan_create(N, C, H, W, F, K, stride, pad, decomp=(0, 0, 0), dtype=DC_BF16, comm=None) -> int:
    out = ctypes.c_void_p()
    _check(lib().dc_plan_create(N, C, H, W, F, K, stride, pad, dc_decomp_t(*decomp), dtype, comm,
                                ctypes.byref(out)))
    return out.value


def dc_plan_create_virtual(N, C, H, W, F, K, stride, pad, decomp, rank, dtype=DC_BF16) -> int:
    out = ctypes.c_void_p()
    _check(lib().dc_plan_create_virtual(N, C, H, W, F, K, stride, pad, dc_decomp_t(*decomp), dtype,
                                        rank, ctypes.byref(out)))
    return out.value


def dc_plan_query(plan: int, t: int) -> dict:
    d = dc_shard_desc_t()
    _check(lib().dc_plan_query(plan, t, ctypes.byref(d)))
    return d.as_dict()


def dc_plan_halo_msgs(plan: int, t: int) -> list[dict]:
    n = ctypes.c_int(0)
    _check(lib().dc_plan_halo_msgs(plan, t, None, ctypes.byref(n)))
    arr = (dc_halo_msg_t * max(n.value, 1))()
    _check(lib().dc_plan_halo_msgs(plan, t, arr, ctypes.byref(n)))
    return [{k: getattr(arr[i], k) for k, _ in dc_halo_msg_t._fields_} for i in range(n.value)]


def dc_plan_decomp(plan: int) -> tuple[tuple[int, int, int], float]:
    d, s = dc_decomp_t(), ctypes.c_double()
    _check(lib().dc_plan_decomp(plan, ctypes.byref(d), ctypes.byref(s)))
    return (d.pn, d.ph, d.pw), s.value


def dc_plan_set_splitk_world(plan: int, world: int):
    """Pick split-K as for the layer divided over `world` ranks (0: the library's basis, the global layer)."""
    _check(lib().dc_plan_set_splitk_world(plan, world))


def dc_plan_destroy(plan: int):
    _check(lib().dc_plan_destroy(plan))


def dc_buffer_alloc(plan: int, t: int) -> int:
    out = ctypes.c_void_p()
    _check(lib().dc_buffer_alloc(plan, t, ctypes.byref(out)))
    return out.value


class _CudaArray:
    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None}


def wrap_device_buffer(ptr: int, shape, dtype=None):
    """Zero-copy torch view of library-owned device memory (e.g. a buffer from
    dc_buffer_alloc) through __cuda_array_interface__. dtype: torch.bfloat16
    (default) or torch.float32."""
    import torch
    dtype = dtype or torch.bfloat16
    if dtype == torch.bfloat16:
        return torch.as_tensor(_CudaArray(ptr, shape, "<u2"), device="cuda").view(torch.bfloat16)
    if dtype == torch.float32:
        return torch.as_tensor(_CudaArray(ptr, shape, "<f4"), device="cuda")
    raise ValueError("dtype must be bfloat16 or float32")


def dc_tensor_import(plan: int, t: int, src, dst, flags: int = 0, stream=None):
    """Owned block of the margined buffer dst from a dense NHWC tensor
    [n][h][w][C] (fp32, or bf16 with DC_SRC_BF16), host or device memory
    (bf16 plans round, fp32 plans store the 3xTF32 hi/lo split)."""
    _check(lib().dc_tensor_import(plan, t, _ptr(src), _ptr(dst), flags, _stream(stream)))


def dc_halo_exchange(plan: int, t: int, buf, flags: int = 0, stream=None):
    _check(lib().dc_halo_exchange(plan, t, _ptr(buf), flags, _stream(stream)))


def dc_conv_fwd(plan: int, x, w, y, flags: int = DC_EXCHANGE, stream=None):
    _check(lib().dc_conv_fwd(plan, _ptr(x), _ptr(w), _ptr(y), flags, _stream(stream)))


def dc_conv_bwd_data(plan: int, dy, w, dx, flags: int = DC_EXCHANGE, stream=None):
    _check(lib().dc_conv_bwd_data(plan, _ptr(dy), _ptr(w), _ptr(dx), flags, _stream(stream)))


def dc_conv_bwd_filter(plan: int, x, dy, dw, flags: int = DC_ALLREDUCE, stream=None):
    _check(lib().dc_conv_bwd_filter(plan, _ptr(x), _ptr(dy), _ptr(dw), flags, _stream(stream)))


def dc_conv_bwd(plan: int, x, dy, w, dx, dw, flags: int = DC_DEFAULT_FLAGS, stream=None):
    _check(lib().dc_conv_bwd(plan, _ptr(x), _ptr(dy), _ptr(w), _ptr(dx), _ptr(dw), flags,
                             _stream(stream)))


def dc_bn_spatial_stats(plan: int, t, mean, var, flags: int = 0, stream=None, local_only: bool = False):
    """flags: DC_BN_LOCAL | DC_BN_FROM_FWD (local_only=True is DC_BN_LOCAL)."""
    flags = int(flags) | (DC_BN_LOCAL if local_only else 0)
    _check(lib().dc_bn_spatial_stats(plan, _ptr(t), _ptr(mean), _ptr(var), flags, _stream(stream)))


def dc_bn_apply(plan: int, y, mean, var, gamma, beta, eps: float = 1e-5, residual=None, flags: int = DC_RELU,
                dst_plan: int | None = None, dst=None, stream=None):
    """out = [relu](BN(y) + residual) into dst (dst_plan's margined input, or dense)."""
    _check(lib().dc_bn_apply(plan, _ptr(y), _ptr(mean), _ptr(var), _ptr(gamma), _ptr(beta), eps, _ptr(residual),
                             flags, dst_plan, _ptr(dst), _stream(stream)))


def dc_bn_backward(plan: int, dout, y, mean, var, gamma, beta, dy_margined, eps: float = 1e-5, residual=None,
                   flags: int = DC_RELU, dgamma=None, dbeta=None, dresidual=None, stream=None):
    """dy (into the owned block of the plan's margined dy buffer), dgamma, dbeta, dresidual."""
    _check(lib().dc_bn_backward(plan, _ptr(dout), _ptr(y), _ptr(mean), _ptr(var), _ptr(gamma), _ptr(beta), eps,
                                _ptr(residual), flags, _ptr(dgamma), _ptr(dbeta), _ptr(dresidual), _ptr(dy_margined),
                                _stream(stream)))


def dc_kernel_launches() -> int:
    return int(lib().dc_kernel_launches())


def dc_model_set_comm(alpha: float, beta: float):
    _check(lib().dc_model_set_comm(alpha, beta))


def dc_model_set_overlap(overlap: bool):
    _check(lib().dc_model_set_overlap(1 if overlap else 0))


def dc_model_set_strided_latency(alpha_w: float):
    _check(lib().dc_model_set_strided_latency(alpha_w))


def dc_model_load_table(path: str):
    _check(lib().dc_model_load_table(path.encode()))


def dc_model_layer_cost(N, C, H, W, F, K, stride, pad, decomp, include_allreduce=True) -> float:
    s = ctypes.c_double()
    _check(lib().dc_model_layer_cost(N, C, H, W, F, K, stride, pad, dc_decomp_t(*decomp),
                                     int(include_allreduce), ctypes.byref(s)))
    return s.value


def dc_model_choose(N, C, H, W, F, K, stride, pad, world) -> tuple[tuple[int, int, int], float]:
    d, s = dc_decomp_t(), ctypes.c_double()
    _check(lib().dc_model_choose(N, C, H, W, F, K, stride, pad, world, ctypes.byref(d), ctypes.byref(s)))
    return (d.pn, d.ph, d.pw), s.value


def dc_model_choose_fixed(N, C, H, W, F, K, stride, pad, world, fix) -> tuple[tuple[int, int, int], float]:
    """Argmin over the grids matching fix's non-zero entries ((1, 0, 0): pure spatial)."""
    d, s = dc_decomp_t(), ctypes.c_double()
    _check(lib().dc_model_choose_fixed(N, C, H, W, F, K, stride, pad, world, dc_decomp_t(*fix), ctypes.byref(d),
                                       ctypes.byref(s)))
    return (d.pn, d.ph, d.pw), s.value


def dc_model_shuffle_cost(N, Ch, H, W, src, dst) -> float:
    """Shuffle(D_i, D_j) of an N x Ch x H x W activation between two grids."""
    t = ctypes.c_double()
    _check(lib().dc_model_shuffle_cost(N, Ch, H, W, dc_decomp_t(*src), dc_decomp_t(*dst), ctypes.byref(t)))
    return t.value


def dc_model_strategy(layers, world: int, fix_pn: int = 0):
    """layers: [(N, C, H, W, F, K, stride, pad, parent[, parent2])]; returns
    ([(pN, pH, pW)] per layer, model seconds)."""
    arr = (dc_layer_t * len(layers))()
    for i, l in enumerate(layers):
        arr[i] = dc_layer_t(*l[:9], l[9] if len(l) > 9 else -1)
    out = (dc_decomp_t * len(layers))()
    t = ctypes.c_double()
    _check(lib().dc_model_strategy(arr, len(layers), world, fix_pn, out, ctypes.byref(t)))
    return [(d.pn, d.ph, d.pw) for d in out], t.value


def dc_redist_create(src_plan: int, src_t: int, dst_plan: int, dst_t: int) -> int:
    """Redistribution (Shuffle) of tensor src_t of src_plan
    into the margined tensor dst_t of dst_plan (collective)."""
    out = ctypes.c_void_p()
    _check(lib().dc_redist_create(src_plan, src_t, dst_plan, dst_t, ctypes.byref(out)))
    return out.value


def dc_redist_bytes(r: int, world: int):
    """([bytes sent to rank q], [bytes received from rank q]) on this rank."""
    snd, rcv = (ctypes.c_int64 * world)(), (ctypes.c_int64 * world)()
    _check(lib().dc_redist_bytes(r, snd, rcv))
    return list(snd), list(rcv)


def dc_redistribute(r: int, src, dst, flags: int = 0, stream=None):
    _check(lib().dc_redistribute(r, _ptr(src), _ptr(dst), flags, _stream(stream)))


def dc_redist_destroy(r: int):
    _check(lib().dc_redist_destroy(r))


def dc_cplan_create(N, C, H, W, F, K, stride, pad, pn: int, pc: int, dtype=DC_BF16, comm=None) -> int:
    """Channel / filter parallel plan on a p_N x p_C grid."""
    out = ctypes.c_void_p()
    _check(lib().dc_cplan_create(N, C, H, W, F, K, stride, pad, pn, pc, dtype, comm, ctypes.byref(out)))
    return out.value


def dc_cplan_create_virtual(N, C, H, W, F, K, stride, pad, pn: int, pc: int, rank: int) -> int:
    out = ctypes.c_void_p()
    _check(lib().dc_cplan_create_virtual(N, C, H, W, F, K, stride, pad, pn, pc, rank, ctypes.byref(out)))
    return out.value


def dc_cplan_query(plan: int, t: int) -> dict:
    """Shard descriptor of t plus "c0", its first global channel."""
    d = dc_shard_desc_t()
    c0 = ctypes.c_int64()
    _check(lib().dc_cplan_query(plan, t, ctypes.byref(d), ctypes.byref(c0)))
    out = d.as_dict()
    out["c0"] = c0.value
    return out


def dc_cconv_fwd(plan: int, x, w, y, flags: int = 0, stream=None):
    _check(lib().dc_cconv_fwd(plan, _ptr(x), _ptr(w), _ptr(y), flags, _stream(stream)))


def dc_cconv_bwd_data(plan: int, dy, w, dx, flags: int = 0, stream=None):
    _check(lib().dc_cconv_bwd_data(plan, _ptr(dy), _ptr(w), _ptr(dx), flags, _stream(stream)))


def dc_cconv_bwd_filter(plan: int, x, dy, dw, flags: int = 0, stream=None):
    _check(lib().dc_cconv_bwd_filter(plan, _ptr(x), _ptr(dy), _ptr(dw), flags, _stream(stream)))


def dc_cplan_destroy(plan: int):
    _check(lib().dc_cplan_destroy(plan))


def dc_pool_create(N, C, H, W, K, stride, pad, decomp, dtype=DC_BF16, comm=None) -> int:
    """Max pooling on a sample x spatial grid."""
    out = ctypes.c_void_p()
    _check(lib().dc_pool_create(N, C, H, W, K, stride, pad, dc_decomp_t(*decomp), dtype, comm, ctypes.byref(out)))
    return out.value


def dc_pool_plans(pool: int):
    """(in_plan, out_plan): x's wide-halo plan, the y / dy / dx plan."""
    a, b = ctypes.c_void_p(), ctypes.c_void_p()
    _check(lib().dc_pool_plans(pool, ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def dc_pool_fwd(pool: int, x, y, flags: int = DC_EXCHANGE, stream=None):
    _check(lib().dc_pool_fwd(pool, _ptr(x), _ptr(y), flags, _stream(stream)))


def dc_pool_bwd(pool: int, x, dy, dx, flags: int = DC_EXCHANGE, stream=None):
    _check(lib().dc_pool_bwd(pool, _ptr(x), _ptr(dy), _ptr(dx), flags, _stream(stream)))


def dc_pool_destroy(pool: int):
    _check(lib().dc_pool_destroy(pool))
