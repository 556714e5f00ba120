// halo.cuh -- halo pack/unpack/P2P copy kernels and BN statistics kernels.
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace dc {

// One strided block copy: nn samples x rows x cols pixels of `vec16` 16-byte
// vectors each (a pixel = c_pad channels), from src to dst (either may be a
// peer-mapped pointer or a contiguous staging buffer).
struct BlockCopy {
    const uint4 *src;
    uint4 *dst;
    long long s_sn, s_sh, s_sw;  // src strides in 16-byte units
    long long d_sn, d_sh, d_sw;  // dst strides in 16-byte units
    int nn, rows, cols, vec16;
};

constexpr int kMaxCopies = 8;
struct CopyBatch {
    BlockCopy c[kMaxCopies];
    int count;
};

// Copies every block of the batch (blockIdx.y = block index). 16-byte
// vectorised, coalesced along the contiguous (col, channel) run.
void launch_block_copies(const CopyBatch &b, cudaStream_t st);

// Stores `value` to each of `n` flags (possibly peer-mapped) with release
// semantics at system scope, after a system-scope fence.
void launch_signal(uint32_t *const *flags, int n, uint32_t value, cudaStream_t st);

// BN statistics of a dense NHWC bf16 tensor [npix][cpad]: per-channel fp64
// sum and sum of squares over all pixels (deterministic two-stage reduce).
// partials must hold blocks * 2 * cpad doubles; out holds 2 * cpad doubles
// (sums then sums of squares).
int bn_partial_blocks(long long npix, int cpad);
// Per-channel sum / sum of squares of an owned NHWC bf16 block into out[2][cpad]
// (fp64, fixed order); with `mean` non-null also mean/var over `count` pixels.
void launch_bn_sums(const __nv_bfloat16 *t, long long npix, int cpad, double *partials,
                    double *out, int c, double count, double *mean, double *var, cudaStream_t st);
// mean = s / count, var = ss / count - mean^2 (biased), first `c` channels.
void launch_bn_finalize(const double *sums, int cpad, int c, double count, double *mean,
                        double *var, cudaStream_t st);

}  // namespace dc

namespace dc {

// One-launch direct P2P halo exchange (epoch e):
//   1. block 0 stores e (release, system scope) into each receiver-side
//      "ready" flag of the peers that send to me  (my margins are free);
//   2. every block waits (acquire polling) until each peer I send to has
//      flagged ready for epoch e;
//   3. all blocks copy the slabs straight into the peers' margins (NVLink);
//   4. each block, after a system fence, atomically adds 1 to the peer's
//      "data" counter for me; a receiver's margin for epoch e is complete when
//      its counter reaches kP2PBlocks * e (waited with cuStreamWaitValue32).
constexpr int kP2PBlocks = 32;
struct P2PExchange {
    CopyBatch copies;
    uint32_t *ready_out[8];  // peers' ready flags for me (I am their receiver)
    uint32_t *ready_in[8];   // my flags written by the peers I send to
    uint32_t *data_out[8];   // peers' data counters for me (I am their sender)
    uint32_t *data_in[8];    // my counters written by the peers that send to me
    int n_ready_out, n_ready_in, n_data_out, n_data_in;
    int wait_in_kernel;      // block 0 polls data_in >= kP2PBlocks*epoch before exiting
    uint32_t epoch;
};
void launch_p2p_exchange(const P2PExchange &x, cudaStream_t st);

}  // namespace dc
