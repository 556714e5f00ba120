// redist.cuh -- redistribution of an activation between two decompositions
// (Shuffle(D_i, D_j)): every rank's owned block under the
// source decomposition is cut along the destination decomposition's owned
// blocks and each piece is stored straight into its new owner's buffer.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dc {

// One piece: nn samples x rows rows of `run` contiguous 16-byte vectors (a row
// of cols pixels of the dense channel vector), from src to dst (dst may be a
// peer's buffer mapped here, or a staging buffer).
struct RedistPiece {
    const uint4 *src;
    uint4 *dst;
    long long s_sn, s_sh;  // src strides (16-byte units) between samples / rows
    long long d_sn, d_sh;  // dst strides
    int nn, rows, run;
};

constexpr int kRedistMaxPeers = 8;
// Blocks of the P2P launch (real ranks; a loopback group uses fewer), the same
// on every rank: a receiver's counter for one sender reaches nblocks * e when
// epoch e has fully arrived.
constexpr int kRedistBlocks = 296;

// One-launch all-to-all over peer memory (epoch e = *epoch_ctr + 1):
//   1. block 0 raises the ready flag (value e) in each sender's flag array:
//      this rank's destination buffer is free (everything the caller queued
//      before on this stream, e.g. the last reader of it, has completed);
//   2. all blocks wait until every receiver has raised its flag for epoch e;
//   3. the pieces are stored into the receivers' buffers (NVLink stores; the
//      piece a rank keeps is a local copy);
//   4. each block adds 1 to every receiver's data counter for this rank after
//      a system fence; block 0 returns when every sender's counter here has
//      reached nblocks * e, so the stream's next kernel sees the data.
struct RedistP2P {
    RedistPiece piece[kRedistMaxPeers];  // one per receiver (this rank included)
    int npiece;
    uint32_t *ready_out[kRedistMaxPeers];  // my ready flag in each sender's array
    uint32_t *ready_in[kRedistMaxPeers];   // receivers' ready flags in my array
    uint32_t *data_out[kRedistMaxPeers];   // my counter in each receiver's array
    uint32_t *data_in[kRedistMaxPeers];    // senders' counters in my array
    int n_ready_out, n_ready_in, n_data_out, n_data_in;
    uint32_t *epoch_ctr;  // {epoch, blocks done} of this redistribution (device)
    int nblocks;          // launch size, equal on every rank
};
void launch_redist_p2p(const RedistP2P &r, cudaStream_t st);

// Plain copies of up to kRedistMaxPeers pieces (NCCL transport: pack into /
// unpack from the staging buffers, and the piece a rank keeps).
void launch_redist_copy(const RedistPiece *pieces, int n, cudaStream_t st);

}  // namespace dc
