// cfpar.cuh -- device protocol of channel / filter parallelism
// (capi.cu dc_cconv_*): the conv GEMMs of the p ranks of a
// channel group store their fp32 partial sums straight into the owners'
// receive slots over peer memory (conv_v2 scatter epilogue); each owner sums
// its p slots in rank order (the reduce of the reduce-scatter).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dc {

constexpr int kCfMaxGroup = 8;

// Flags of one exchange, epoch e = *epoch + 1 (device, graph-replayable).
struct CfFlags {
    uint32_t *out[kCfMaxGroup];       // my flag in each peer's array
    const uint32_t *in[kCfMaxGroup];  // peers' flags in my array
    int n;                            // flags in `out` (and in `in`, unless n_in > 0)
    int n_in;                         // flags in `in` when it differs from n (0: n)
    uint32_t *epoch;                  // {epoch, blocks done}
    int publish;                      // launch_cf_wait: publish epoch e when done
};

// One block: raise my flag (value e) in every peer's array, then wait until
// every peer's flag in my array reached e. With the "ready" arrays: this
// rank's receive slots are free (everything queued before on the stream has
// completed) and every owner's slots are free, so the GEMM may store.
void launch_cf_handshake(const CfFlags &f, cudaStream_t st);
// One block: wait until every peer's flag in my array reached e (the
// senders' "data" flags, raised by launch_signal after their GEMMs); with
// `publish`, then advance the epoch.
void launch_cf_wait(const CfFlags &f, cudaStream_t st);

// out[pix][c] = bf16( sum_{s = 0..n-1} slots[s][pix][c] ) for c < seg (fixed
// rank order); slot s starts slot_stride floats after slot s - 1 and holds
// npix x seg fp32; out channel pitch out_pitch.
// The last block publishes the epoch (epoch[0] = epoch[0] + 1).
void launch_cf_reduce(const float *slots, int n, long long slot_stride, long long npix, int seg, void *out,
                      int out_pitch, uint32_t *epoch, cudaStream_t st);

}  // namespace dc
