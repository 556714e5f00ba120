// redist.cu -- the redistribution (Shuffle) kernels: the
// one-launch all-to-all over peer memory and the plain piece copies of the
// NCCL transport (redist.cuh).
//
// A piece is nn x rows runs of `run` contiguous 16-byte vectors (the pixels of
// one row of the intersection block, every channel): one warp moves one run,
// four vectors per lane in flight, so every load and store is a coalesced
// 512-byte warp access whether the destination is local or a peer's buffer
// mapped over NVLink.
#include "common.hpp"
#include "launch.cuh"
#include "redist.cuh"

namespace dc {

namespace {

__device__ __forceinline__ void copy_run(const uint4 *__restrict__ s, uint4 *__restrict__ d, int run, int lane) {
    int v = lane;
    for (; v + 96 < run; v += 128) {
        const uint4 a = s[v], b = s[v + 32], c = s[v + 64], e = s[v + 96];
        d[v] = a, d[v + 32] = b, d[v + 64] = c, d[v + 96] = e;
    }
    for (; v < run; v += 32) d[v] = s[v];
}

// Grid-stride over the runs of all pieces, one warp per run.
__device__ __forceinline__ void copy_pieces(const RedistPiece *pieces, int n) {
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    const long long w0 = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    for (int k = 0; k < n; ++k) {
        const RedistPiece &p = pieces[k];
        const long long runs = (long long)p.nn * p.rows;
        for (long long i = w0; i < runs; i += warps) {
            const int s = (int)(i / p.rows), r = (int)(i - (long long)s * p.rows);
            copy_run(p.src + s * p.s_sn + r * p.s_sh, p.dst + s * p.d_sn + r * p.d_sh, p.run, lane);
        }
    }
}

__global__ void __launch_bounds__(256) redist_p2p_kernel(const __grid_constant__ RedistP2P x) {
    pdl_wait();  // (launch.cuh: PDL)
    const uint32_t e = *reinterpret_cast<volatile uint32_t *>(x.epoch_ctr) + 1;
    if (blockIdx.x == 0 && (int)threadIdx.x < x.n_ready_out) {
        __threadfence_system();
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(x.ready_out[threadIdx.x]), "r"(e) : "memory");
    }
    if ((int)threadIdx.x < x.n_ready_in) spin_until_geq(x.ready_in[threadIdx.x], e);
    __syncthreads();
    copy_pieces(x.piece, x.npiece);
    __syncthreads();
    if ((int)threadIdx.x < x.n_data_out) {
        __threadfence_system();
        atomicAdd_system(x.data_out[threadIdx.x], 1u);
    }
    if (blockIdx.x == 0 && (int)threadIdx.x < x.n_data_in) {
        spin_until_geq(x.data_in[threadIdx.x], (uint32_t)x.nblocks * e);
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

struct PieceBatch {
    RedistPiece piece[kRedistMaxPeers];
    int n;
};

__global__ void __launch_bounds__(256) redist_copy_kernel(const __grid_constant__ PieceBatch b) {
    pdl_wait();  // (launch.cuh: PDL)
    copy_pieces(b.piece, b.n);
}

}  // namespace

void launch_redist_p2p(const RedistP2P &r, cudaStream_t st) {
    launch_k(redist_p2p_kernel, dim3(r.nblocks), dim3(256), 0, st, 1, "redist p2p", r);
}

void launch_redist_copy(const RedistPiece *pieces, int n, cudaStream_t st) {
    DC_REQUIRE(n >= 0 && n <= kRedistMaxPeers, DC_ERR_ARG, "redist copy: %d pieces", n);
    PieceBatch b{};
    long long runs = 0;
    for (int k = 0; k < n; ++k) {
        b.piece[b.n++] = pieces[k];
        runs += (long long)pieces[k].nn * pieces[k].rows;
    }
    if (runs == 0) return;
    const int blocks = (int)std::min<long long>((runs + 7) / 8, kRedistBlocks);
    launch_k(redist_copy_kernel, dim3(blocks), dim3(256), 0, st, 1, "redist copy", b);
}

// (CUDA lazy loading: see preload_halo)
void preload_redist() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(redist_p2p_kernel));
    cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(redist_copy_kernel));
}

}  // namespace dc
