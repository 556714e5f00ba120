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
// value = *epoch_src + 1 when epoch_src is set (device epoch, graph-replayable)
void launch_signal(uint32_t *const *flags, int n, uint32_t value, const uint32_t *epoch_src, cudaStream_t st);

// Fixed-order reduction of `blocks` partials [blocks][2][cpad] into out[2][cpad]
// (+ mean / var when `mean` is set): the fused forward-epilogue partials, or
// those of the staged pass (bn.cuh launch_bn_stats).
void launch_bn_reduce(const double *partials, int blocks, int cpad, double *out, int c, double count, double *mean,
                      double *var, cudaStream_t st);
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
    // device epoch of this (plan, buffer): {epoch, blocks done}. Every block
    // reads epoch + 1 at start; the last block to finish publishes it and
    // resets the count (so the launch can be replayed from a CUDA graph; the
    // fused conv_v2 exchange uses the same words). Each epoch adds kP2PBlocks
    // to every receiver's data counter (32 blocks, or 32 slices when fused).
    uint32_t *epoch_ctr;
};
void launch_p2p_exchange(const P2PExchange &x, cudaStream_t st);

// ---------------------------------------------------------------------------
// Spatial BN statistics allreduce over NVLink (one kernel, one block): every
// member of the plan's BN group stores its 2*cpad fp64 sums into slot
// [parity][its index] of every member's mailbox (peer memory mapped through
// CUDA IPC, or plain pointers in a loopback group), raises its flag to the
// epoch, waits for all members' flags, and sums the slots in member order
// (deterministic, identical on every member). The epoch lives on the device
// (read at start, published at the end) so the kernel can be replayed from a
// CUDA graph. The mailbox belongs to ONE plan, whose members all take part in
// every epoch, so a member is at most one epoch ahead of any other (it needs
// everyone's flag to finish) and two alternating parities suffice.
// ---------------------------------------------------------------------------
constexpr int kMaxBnGroup = 8;

struct BnP2P {
    double *peer_box[kMaxBnGroup];      // member k's mailbox data (mapped)
    uint32_t *peer_flags[kMaxBnGroup];  // member k's flag array (mapped)
    const double *my_box;               // my mailbox data
    const uint32_t *my_flags;           // my flag array (flag k: member k's epoch)
    int gsize, my_idx;                  // members, my index in the group
    uint32_t *epoch;                    // device epoch counter (this plan)
    const double *local;                // my 2 * cpad sums
    int cpad, c;
    double count;
    double *sums;                       // out: global sums [2 * cpad]
    double *mean, *var;                 // out: first c channels
};
void launch_bn_allreduce_p2p(const BnP2P &b, cudaStream_t st);

}  // namespace dc
