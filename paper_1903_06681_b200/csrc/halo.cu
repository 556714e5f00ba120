// halo.cu -- halo slab copies and the
// spatially-aggregated BN statistics kernels.
//
// In NHWC a halo slab of an H split is, per sample, a contiguous run of
// rows*wb*c_pad elements; a W split slab is `rows` runs of cols*c_pad. One
// kernel handles both: each thread moves one 16-byte vector, consecutive
// threads walk the contiguous (col, channel) run, so loads and stores are
// fully coalesced whether the destination is local staging (NCCL baseline)
// or a neighbour's margin mapped over NVLink (direct P2P stores).
#include "common.hpp"
#include "halo.cuh"
#include "launch.cuh"

namespace dc {

__global__ void block_copy_kernel(const CopyBatch b) {
    pdl_wait();  // (launch.cuh: PDL)
    const BlockCopy &c = b.c[blockIdx.y];
    const long long run = (long long)c.cols * c.vec16;        // vectors per (n, row)
    const long long total = (long long)c.nn * c.rows * run;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long nr = idx / run, k = idx - nr * run;
        const int n = (int)(nr / c.rows), r = (int)(nr - (long long)n * c.rows);
        const int col = (int)(k / c.vec16), v = (int)(k - (long long)col * c.vec16);
        const uint4 val = c.src[n * c.s_sn + r * c.s_sh + col * c.s_sw + v];
        c.dst[n * c.d_sn + r * c.d_sh + col * c.d_sw + v] = val;
    }
}

void launch_block_copies(const CopyBatch &b, cudaStream_t st) {
    if (b.count == 0) return;
    long long mx = 0;
    for (int i = 0; i < b.count; ++i)
        mx = std::max(mx, (long long)b.c[i].nn * b.c[i].rows * b.c[i].cols * b.c[i].vec16);
    if (mx == 0) return;
    const int blocks = (int)std::min<long long>((mx + 255) / 256, 148 * 4);
    launch_k(block_copy_kernel, dim3(blocks, b.count), dim3(256), 0, st, 1, "block copy", b);
}

struct FlagList {
    uint32_t *f[16];
};

__global__ void signal_kernel(FlagList fl, int n, uint32_t value, const uint32_t *epoch_src) {
    pdl_wait();  // (launch.cuh: PDL)
    if (epoch_src) value = *reinterpret_cast<const volatile uint32_t *>(epoch_src) + 1;
    __threadfence_system();
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(fl.f[i]), "r"(value) : "memory");
}

void launch_signal(uint32_t *const *flags, int n, uint32_t value, const uint32_t *epoch_src, cudaStream_t st) {
    if (n == 0) return;
    DC_REQUIRE(n <= 16, DC_ERR_ARG, "too many flags");
    FlagList fl{};
    for (int i = 0; i < n; ++i) fl.f[i] = flags[i];
    launch_k(signal_kernel, dim3(1), dim3(32), 0, st, 1, "signal", fl, n, value, epoch_src);
}

// ---------------------------------------------------------------------------
// BN statistics: the per-block partial sums come from the staged pass
// (bn.cu, bn_staged_kernel<kBnStats>) or the fused conv epilogue.
// ---------------------------------------------------------------------------
// Fixed-order reduction of the per-block partials (deterministic).
// One warp per output value: lane l sums the partials of blocks l, l+32, ...
// in that order, loading 8 of them at a time (independent loads in flight),
// then a fixed xor-shuffle tree. With `mean` set, lane 0 of the warps of
// channel i also finalises mean/var (the single-group case: no allreduce).
__global__ void bn_reduce_kernel(const double *__restrict__ partials, int blocks, int cpad,
                                 double *__restrict__ out, int c, double count,
                                 double *__restrict__ mean, double *__restrict__ var) {
    pdl_wait();  // (launch.cuh: PDL)
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int n2 = 2 * cpad;
    if (warp >= cpad) return;
    // warp w reduces sum (w) and sum of squares (cpad + w) of channel w
    double acc[2] = {0.0, 0.0};
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int col = warp + k * cpad;
        int b = lane;
        for (; b + 32 * 7 < blocks; b += 32 * 8) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldg(&partials[(long long)(b + 32 * u) * n2 + col]);
#pragma unroll
            for (int u = 0; u < 8; ++u) acc[k] += v[u];
        }
        for (; b < blocks; b += 32) acc[k] += __ldg(&partials[(long long)b * n2 + col]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
    }
    if (lane == 0) {
        out[warp] = acc[0];
        out[cpad + warp] = acc[1];
        if (mean && warp < c) {
            const double mu = acc[0] / count;
            const double v = acc[1] / count - mu * mu;
            mean[warp] = mu;
            var[warp] = v > 0.0 ? v : 0.0;
        }
    }
}

void launch_bn_reduce(const double *partials, int blocks, int cpad, double *out, int c, double count, double *mean,
                      double *var, cudaStream_t st) {
    launch_k(bn_reduce_kernel, dim3((cpad * 32 + 255) / 256), dim3(256), 0, st, 1, "bn reduce", partials, blocks,
             cpad, out, c, count, mean, var);
}

__global__ void bn_finalize_kernel(const double *sums, int cpad, int c, double count, double *mean,
                                   double *var) {
    pdl_wait();  // (launch.cuh: PDL)
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < c; i += gridDim.x * blockDim.x) {
        const double mu = sums[i] / count;
        const double v = sums[cpad + i] / count - mu * mu;
        mean[i] = mu;
        var[i] = v > 0.0 ? v : 0.0;
    }
}

void launch_bn_finalize(const double *sums, int cpad, int c, double count, double *mean,
                        double *var, cudaStream_t st) {
    launch_k(bn_finalize_kernel, dim3((c + 255) / 256), dim3(256), 0, st, 1, "bn finalize", sums, cpad, c, count,
             mean, var);
}

}  // namespace dc

namespace dc {

__global__ void __launch_bounds__(256) p2p_exchange_kernel(const __grid_constant__ P2PExchange x) {
    pdl_wait();  // (launch.cuh: PDL)
    const uint32_t e = *reinterpret_cast<volatile uint32_t *>(x.epoch_ctr) + 1;
    if (blockIdx.x == 0 && (int)threadIdx.x < x.n_ready_out) {
        __threadfence_system();
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(x.ready_out[threadIdx.x]), "r"(e) : "memory");
    }
    if ((int)threadIdx.x < x.n_ready_in) spin_until_geq(x.ready_in[threadIdx.x], e);
    __syncthreads();
    for (int k = 0; k < x.copies.count; ++k) {
        const BlockCopy &c = x.copies.c[k];
        const long long run = (long long)c.cols * c.vec16;
        const long long total = (long long)c.nn * c.rows * run;
        for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
             idx += (long long)gridDim.x * blockDim.x) {
            const long long nr = idx / run, kk = idx - nr * run;
            const int n = (int)(nr / c.rows), r = (int)(nr - (long long)n * c.rows);
            const int col = (int)(kk / c.vec16), v = (int)(kk - (long long)col * c.vec16);
            c.dst[n * c.d_sn + r * c.d_sh + col * c.d_sw + v] = c.src[n * c.s_sn + r * c.s_sh + col * c.s_sw + v];
        }
    }
    __syncthreads();
    if ((int)threadIdx.x < x.n_data_out) {
        __threadfence_system();
        atomicAdd_system(x.data_out[threadIdx.x], 1u);
    }
    // block 0 returns only when every sender's blocks have delivered epoch e
    if (blockIdx.x == 0 && (int)threadIdx.x < x.n_data_in) {
        spin_until_geq(x.data_in[threadIdx.x], kP2PBlocks * e);
        __threadfence_system();
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // the last block publishes the epoch and resets the count
        const uint32_t prev = atomicAdd(x.epoch_ctr + 1, 1u);
        if (prev == gridDim.x - 1) {
            x.epoch_ctr[1] = 0;
            __threadfence();
            *reinterpret_cast<volatile uint32_t *>(x.epoch_ctr) = e;
        }
    }
}

void launch_p2p_exchange(const P2PExchange &x, cudaStream_t st) {
    launch_k(p2p_exchange_kernel, dim3(kP2PBlocks), dim3(256), 0, st, 1, "p2p exchange", x);
}

__global__ void __launch_bounds__(256) bn_allreduce_p2p_kernel(const __grid_constant__ BnP2P b) {
    pdl_wait();  // (launch.cuh: PDL)
    const uint32_t e = *reinterpret_cast<volatile uint32_t *>(b.epoch) + 1;
    const int par = e & 1;
    const int n2 = 2 * b.cpad;
    const long long slot = n2;
    const long long par_stride = (long long)b.gsize * slot;
    // 1. my sums into slot [par][my_idx] of every member (me included)
    for (int k = 0; k < b.gsize; ++k) {
        double *dst = b.peer_box[k] + par * par_stride + b.my_idx * slot;
        for (int i = threadIdx.x; i < n2; i += blockDim.x) dst[i] = b.local[i];
    }
    __threadfence_system();
    __syncthreads();
    if ((int)threadIdx.x < b.gsize)
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(b.peer_flags[threadIdx.x] + b.my_idx), "r"(e)
                     : "memory");
    // 2. wait until every member has delivered epoch e
    if ((int)threadIdx.x < b.gsize) spin_until_geq(b.my_flags + threadIdx.x, e);
    __syncthreads();
    // 3. fixed-order sum over the members (uncached loads: peers wrote them)
    for (int i = threadIdx.x; i < n2; i += blockDim.x) {
        double acc = 0.0;
        for (int k = 0; k < b.gsize; ++k) acc += __ldcv(b.my_box + par * par_stride + k * slot + i);
        b.sums[i] = acc;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < b.c; i += blockDim.x) {
        const double mu = b.sums[i] / b.count;
        const double v = b.sums[b.cpad + i] / b.count - mu * mu;
        b.mean[i] = mu;
        b.var[i] = v > 0.0 ? v : 0.0;
    }
    if (threadIdx.x == 0) *reinterpret_cast<volatile uint32_t *>(b.epoch) = e;
}

void launch_bn_allreduce_p2p(const BnP2P &b, cudaStream_t st) {
    DC_REQUIRE(b.gsize <= kMaxBnGroup, DC_ERR_UNSUPPORTED, "P2P BN allreduce: too many members");
    launch_k(bn_allreduce_p2p_kernel, dim3(1), dim3(256), 0, st, 1, "bn p2p", b);
}


// Loads this file's kernels now (CUDA lazy loading would otherwise load a
// kernel at its first launch, which waits for the device: with the spinning
// halo / BN protocol kernels of a loopback group in flight, that wait never
// ends).
void preload_halo() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(block_copy_kernel));
    cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(signal_kernel));
    cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(bn_reduce_kernel));
    cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(bn_finalize_kernel));
    cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(p2p_exchange_kernel));
    cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(bn_allreduce_p2p_kernel));
}

}  // namespace dc
