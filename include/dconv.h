/*
 * dconv.h -- C ABI of the B200-native spatially / hybrid sample-spatial
 * partitioned 2D convolution library (libdconv.so), after Dryden et al.,
 * "Improving Strong-Scaling of CNN Training by Exploiting Finer-Grained
 * Parallelism", arXiv:1903.06681 (cited below as PAPER.md:<line>).
 *
 * One process per GPU. Every tensor argument is a plain device pointer
 * unless stated; every size is in elements. No torch types cross this ABI.
 *
 * Problem: input x N x C x H x W, weights w F x C x K x K,
 * output y N x F x Ho x Wo with stride S and padding P,
 *   Ho = floor((H + 2P - K)/S) + 1   (reading R2).
 * The operation is cross-correlation, Eq. 1 (reading R1).
 *
 * Device layouts:
 *   activations  NHWC bf16, channels padded to c_pad = roundup(C, 16)
 *                (padded channels must be zero); x and dy live in
 *                "margined" buffers [n][hb][wb][c_pad] holding the owned
 *                block plus the halo rows/cols from the neighbours;
 *   y, dx        dense NHWC bf16 over the owned block [n][h][w][c_pad];
 *   w            bf16 [F][K][K][c_pad(C)]  (replicated on every rank,
 *                PAPER.md:137 "w and dL/dw are replicated");
 *   dw           fp32 [F][K][K][C]  (dense, no channel padding: the F C K^2
 *                words the allreduce sends).
 *
 * Semantics: every call enqueues work on the caller's stream and returns
 * without a host sync; internal streams are joined back with events before
 * returning. Calls marked COLLECTIVE must be made by all ranks of the comm
 * in the same order (as in NCCL). A plan is not thread-safe; distinct plans
 * are independent. Nothing is thrown across the ABI: every entry point
 * returns a dc_status_t and dc_last_error() gives a thread-local message.
 */
#ifndef DCONV_H
#define DCONV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    DC_OK = 0,
    DC_ERR_ARG = 1,          /* null pointer, bad enum, bad flag             */
    DC_ERR_SHAPE = 2,        /* even K, P > K/2, non-positive extent, ...     */
    DC_ERR_PARTITION = 3,    /* grid invalid for the shape     */
    DC_ERR_UNSUPPORTED = 4,  /* valid but not implemented (e.g. stride > 2)   */
    DC_ERR_CUDA = 5,         /* CUDA failure; the plan becomes unusable       */
    DC_ERR_COMM = 6,         /* NCCL / IPC failure; the plan becomes unusable */
    DC_ERR_OOM = 7
} dc_status_t;

/* Arithmetic of a plan (reading R18; "single-precision"):
 *   DC_BF16        bf16 activations / weights, fp32 accumulation (kind::f16);
 *   DC_FP32_3XTF32 fp32 activations / weights, computed as three tf32
 *                  products per term (x_hi w_hi + x_hi w_lo + x_lo w_hi,
 *                  kind::tf32, fp32 accumulation): ~2^-21 relative error per
 *                  product. Layouts of an fp32 plan: channels padded to a
 *                  multiple of 8; the margined x / dy buffers hold each pixel
 *                  as [hi (c_pad/2) | lo (c_pad/2)] fp32 (fill them with
 *                  dc_tensor_import); y / dx plain fp32 [n][h][w][c_pad];
 *                  w fp32 [F][K][K][c_pad]; dw fp32 [F][K][K][C]. */
typedef enum { DC_BF16 = 0, DC_FP32_3XTF32 = 1 } dc_dtype_t;

typedef enum { DC_X = 0, DC_Y = 1, DC_DY = 2, DC_DX = 3, DC_W = 4, DC_DW = 5 } dc_tensor_t;

/* Process grid (p_N, p_H, p_W); rank = (i_N * p_H + i_H) * p_W + i_W
 * (row-major, reading R8). {0,0,0} asks the performance model to choose
 * (per layer). */
typedef struct { int32_t pn, ph, pw; } dc_decomp_t;

/* Local shard of one tensor on this rank (dc_plan_query). */
typedef struct {
    int64_t n0, h0, w0;         /* global offset of the owned block (samples, rows, cols)   */
    int64_t n, h, w;            /* owned extents                                            */
    int64_t c, c_pad;           /* logical channels, padded channels (innermost)           */
    int32_t halo_n, halo_s;     /* margin rows above / below the owned block (x, dy only)  */
    int32_t halo_w, halo_e;     /* margin cols left / right of the owned block             */
    int64_t hb, wb;             /* buffer extents: hb = halo_n + h + halo_s, wb likewise    */
    int64_t stride_n, stride_h, stride_w; /* element strides of the buffer (stride_c = 1)   */
    size_t bytes;               /* bytes the caller must provide                            */
} dc_shard_desc_t;

typedef struct dc_comm_s *dc_comm_t;
typedef struct dc_plan_s *dc_plan_t;

/* ---- flags ---- */
#define DC_EXCHANGE      0x1u  /* conv_fwd / conv_bwd_data: do the halo exchange inside the
                                  call, overlapped with the interior tiles  */
#define DC_ALLREDUCE     0x2u  /* conv_bwd_filter: sum dW over all ranks    */
#define DC_HALO_NCCL     0x4u  /* use grouped ncclSend/ncclRecv instead of direct P2P       */
#define DC_BN_STATS      0x10u /* conv_fwd: accumulate the BN statistics of the stored y in
                                  the epilogue (per-CTA fp64 partials), reduced by a
                                  following dc_bn_spatial_stats(..., DC_BN_FROM_FWD) on
                                  that unchanged y instead of re-reading it */
#define DC_DETERMINISTIC 0x20u /* accepted for compatibility: dW is deterministic by
                                  default (split-K partials summed in a fixed order) */
#define DC_DW_ATOMIC     0x40u /* conv_bwd_filter / conv_bwd: let the split-K partials of
                                  small dW (< 1M elements) add into dW with fp32 atomics
                                  (no partial buffer / reduce launch; last-bit
                                  differences between runs). y and dx are always
                                  reproducible. */
#define DC_ALLREDUCE_ASYNC 0x8u /* with DC_ALLREDUCE: queue the dW allreduce on the
                                  communicator's gradient stream instead of joining it
                                  into the call (overlaps the later layers' work,
                                  PAPER.md:204, 214); dW is final after dc_comm_sync */
#define DC_NO_OVERLAP    0x80u /* with DC_EXCHANGE (conv_fwd / conv_bwd_data): finish the halo
                                  exchange on the caller's stream, then compute the whole
                                  shard in one pass -- the non-overlapped schedule of the
                                  performance model (no overlap)      */
#define DC_FORCE_OVERLAP 0x100u /* with DC_EXCHANGE: always run the interior tiles while the
                                  halo arrives and the boundary tiles after it.
                                  Default: that overlap only for halos of >= 8 MB per rank;
                                  smaller ones are exchanged first and the shard computed in
                                  one launch (measured faster) */
#define DC_DEFAULT_FLAGS (DC_EXCHANGE | DC_ALLREDUCE)

/* COLLECTIVE. Create the communicator of `world` ranks. nccl_uid128 points to
 * the 128-byte ncclUniqueId produced by dc_comm_unique_id on rank 0 and
 * broadcast by the caller (e.g. through torch.distributed). world == 1
 * needs no id (may be NULL). cuda_device is this rank's device ordinal.
 * Every plan of the communicator shares its few side streams (exchanges,
 * stride phases, imports, the dW allreduces); run the process with
 * CUDA_DEVICE_MAX_CONNECTIONS >= 16 so that they do not alias onto one
 * hardware queue with the caller's streams (bench.py sets 32).
 * Errors: DC_ERR_ARG (rank/world), DC_ERR_COMM (NCCL). */
dc_status_t dc_comm_create(int rank, int world, const void *nccl_uid128, int cuda_device,
                           dc_comm_t *out);
/* NOT collective. Loopback group: `world` virtual ranks (1..64) of THIS
 * process on ONE device (cuda_device), written to comms[0..world-1]. Every
 * call a real rank would make is made once per virtual rank, each on its own
 * stream (host calls never block, so one thread can issue rank 0, 1, ... in
 * turn; the device-side P2P protocols let the ranks' kernels rendezvous).
 * The halo exchange (direct P2P stores, flags, interior/boundary overlap) and
 * the spatial BN mailbox run unchanged with plain pointers in place of
 * IPC-mapped peer memory; the NCCL transports (DC_HALO_NCCL, the dW
 * allreduce, BN groups > 8) need real ranks and fail with
 * DC_ERR_UNSUPPORTED. Used to test the multi-rank device protocols on one
 * GPU. Each virtual rank owns two streams (dc_comm_stream: the one to issue
 * its calls on; the other carries its exchanges), created so that no two
 * ranks share a hardware queue: needs CUDA_DEVICE_MAX_CONNECTIONS >= 2 world
 * in the environment before CUDA initializes (DC_ERR_ARG otherwise; default
 * 8, i.e. up to 4 ranks). Destroy each with dc_comm_destroy.
 * Errors: DC_ERR_ARG, DC_ERR_CUDA. */
dc_status_t dc_comm_create_local(int world, int cuda_device, dc_comm_t *comms);
/* The compute stream of a loopback rank (cudaStream_t): issue that rank's
 * calls on it. Errors: DC_ERR_ARG (not a loopback communicator). */
dc_status_t dc_comm_stream(dc_comm_t comm, void **stream);
/* Write a fresh 128-byte ncclUniqueId to uid128 (rank 0 only). */
dc_status_t dc_comm_unique_id(void *uid128);
dc_status_t dc_comm_destroy(dc_comm_t comm);
/* Make `stream` wait for every dW allreduce queued with DC_ALLREDUCE_ASYNC on
 * this communicator since the previous dc_comm_sync (an event wait: does not
 * block the host; may be recorded into a CUDA graph, in the same capture as
 * the queuing calls). Nothing queued, or world == 1: no-op. */
dc_status_t dc_comm_sync(dc_comm_t comm, void *stream);
/* Bucketing of the DC_ALLREDUCE_ASYNC dW allreduces: the
 * layers' dW buffers are collected until `bytes` (default 4 MiB) and issued
 * as one grouped NCCL call on the gradient stream (after the work queued on
 * the caller's stream so far); dc_comm_sync issues what is left. 0 issues
 * every allreduce at its call. The buffers must not change until
 * dc_comm_sync. Host only. Errors: DC_ERR_ARG. */
dc_status_t dc_comm_set_bucket_bytes(dc_comm_t comm, size_t bytes);

/* COLLECTIVE. Plan one convolution layer: global N, C, H, W, F, odd K,
 * stride in {1, 2}, pad 0 <= P <= K/2, grid `decomp` (product == world, or
 * {0,0,0} for the model's choice -- PAPER.md:206, 222 -- or some entries 0:
 * the model chooses those with the others fixed, e.g. {1,0,0} = the best pure
 * spatial grid), on `comm`.
 * Computes the blocked splits, the owned output blocks, the
 * per-side halo widths of x and dy from the interval formula (PAPER.md:139,
 * 145; reading R5) and validates the partition.
 * Errors: DC_ERR_SHAPE (even K, P > K/2, extent < K without padding),
 * DC_ERR_PARTITION (p_N > N, a part with no output rows, a halo wider than the
 * adjacent rank's block -- PAPER.md:145's degenerate case -- or product !=
 * world), DC_ERR_UNSUPPORTED (stride > 2), DC_ERR_ARG (unknown dtype). */
dc_status_t dc_plan_create(int64_t N, int64_t C, int64_t H, int64_t W, int64_t F, int K,
                           int stride, int pad, dc_decomp_t decomp, dc_dtype_t dtype,
                           dc_comm_t comm, dc_plan_t *out);
/* NOT collective. Plan of rank `rank` of a virtual grid without a
 * communicator: index math only (dc_plan_query / dc_plan_halo_msgs /
 * dc_plan_decomp work; compute calls need decomp product 1). Used by the
 * host-side tests and by the replica mode of bench.py. */
dc_status_t dc_plan_create_virtual(int64_t N, int64_t C, int64_t H, int64_t W, int64_t F, int K,
                                   int stride, int pad, dc_decomp_t decomp, dc_dtype_t dtype,
                                   int rank, dc_plan_t *out);

/* One halo message of this rank (global rows [row0, row0+rows) x cols
 * [col0, col0+cols), all local samples and channels). */
typedef struct {
    int32_t peer;       /* the other rank                                        */
    int32_t is_send;    /* 1: this rank sends the block, 0: it receives it       */
    int64_t row0, rows, col0, cols;
} dc_halo_msg_t;
/* Messages of the x (t = DC_X, before forward) or dy (t = DC_DY, before
 * backward-data) exchange. *count is in/out: capacity in, number out. */
dc_status_t dc_plan_halo_msgs(dc_plan_t plan, dc_tensor_t t, dc_halo_msg_t *msgs, int *count);

/* Shard descriptor of `t` on this rank (sizes the caller must allocate). */
dc_status_t dc_plan_query(dc_plan_t plan, dc_tensor_t t, dc_shard_desc_t *desc);
/* The grid in use and the model's predicted seconds for fwd+bwd of the layer
 * (PAPER.md:206 Cost_D(l)); predicted may be NULL. */
dc_status_t dc_plan_decomp(dc_plan_t plan, dc_decomp_t *chosen, double *predicted_seconds);
/* Summation-order setting of the conv kernels: the split-K factor over
 * channel groups (the only choice that changes how an output is summed) is
 * picked for the global layer divided over `world` ranks. Default (world 0):
 * 1, i.e. from the undivided global layer whatever the plan's grid, so every
 * partition of the layer and its 1-GPU plan sum every y / dx element in the
 * same order (bit-identical outputs, north_star). Plans with equal settings
 * agree bit for bit; another setting trades that for splits fitted to one
 * grid size. Host only; takes effect from the next compute call. */
dc_status_t dc_plan_set_splitk_world(dc_plan_t plan, int world);
dc_status_t dc_plan_destroy(dc_plan_t plan);

/* COLLECTIVE. Allocate (and zero) the margined buffer of t in {DC_X, DC_DY}
 * with cudaMalloc and map it into the neighbours' address spaces for direct
 * P2P halo stores; or (t in {DC_Y, DC_DX}, not collective) a dense shard
 * buffer that a redistribution may target (dc_redist_create maps it into the
 * senders). Owned by the plan; freed by dc_plan_destroy. */
dc_status_t dc_buffer_alloc(dc_plan_t plan, dc_tensor_t t, void **dev_ptr);

/* Fill the OWNED block of a margined buffer (t in {DC_X, DC_DY}, dst from
 * dc_buffer_alloc or any buffer of that layout) from `src`, a dense NHWC
 * tensor of the owned block [n][h][w][C] (C = the tensor's logical channels,
 * no padding) in fp32 -- or bf16 with DC_SRC_BF16 (bf16 plans only) -- in
 * HOST memory (pinned or pageable: one H2D copy into plan-owned staging) or
 * device memory. bf16 plans round fp32 to bf16; fp32 plans store the exact
 * 3xTF32 split [hi | lo] (x_hi = x with its low 13 mantissa bits cleared,
 * x_lo = x - x_hi); padded channels are written as zeros, the margins are
 * left alone (dc_halo_exchange fills them). With DC_IMPORT_ASYNC the copy and
 * the layout kernel run on the plan's copy stream after the work queued on
 * `stream` so far, and the plan's next call that reads that buffer waits for
 * them (so a step can issue every layer's input copy up front and overlap it
 * with compute); otherwise stream-ordered on `stream`. A host src must stay
 * valid until the copy ran. Errors: DC_ERR_ARG. */
#define DC_IMPORT_ASYNC 0x1u
#define DC_SRC_BF16     0x2u
dc_status_t dc_tensor_import(dc_plan_t plan, dc_tensor_t t, const void *src, void *dst, unsigned flags,
                             void *stream);

/* COLLECTIVE. Halo exchange of buffer `buf` (t in {DC_X, DC_DY}): copies each
 * rank's boundary slabs (all local samples and channels) into the
 * neighbours' margins, the 8 neighbours of a 2D grid directly (PAPER.md:127,
 * 137-141, 193-194). Bit-exact copy; positions outside the global tensor are
 * never sent (they are zero padding). flags: DC_HALO_NCCL selects the NCCL
 * send/recv baseline, otherwise direct P2P stores over NVLink.
 * buf must be the pointer returned by dc_buffer_alloc for t. */
dc_status_t dc_halo_exchange(dc_plan_t plan, dc_tensor_t t, void *buf, unsigned flags,
                             void *stream);

/* Forward (Eq. 1 on the owned outputs): y = conv(x, w).
 * x_margined: DC_X buffer (from dc_buffer_alloc when world > 1 and a halo
 * exists; any buffer of the DC_X layout otherwise); w: DC_W; y: DC_Y.
 * With DC_EXCHANGE the x halo exchange runs concurrently with the interior
 * tiles and the boundary tiles run after it. */
dc_status_t dc_conv_fwd(dc_plan_t plan, void *x_margined, const void *w, void *y,
                        unsigned flags, void *stream);

/* Backward-data (Eq. 3 on the owned inputs): dx = conv^T(dy, w).
 * dy_margined: DC_DY buffer; w: DC_W; dx: DC_DX. DC_EXCHANGE as above. */
dc_status_t dc_conv_bwd_data(dc_plan_t plan, void *dy_margined, const void *w, void *dx,
                             unsigned flags, void *stream);

/* Backward-filter (Eq. 2 restricted to the owned outputs):
 * dw = sum over owned (n, i, j) of dy * x, using the halo'd x retained from
 * the forward call (its margins must be unchanged since dc_conv_fwd) and dy
 * WITHOUT its halo. With DC_ALLREDUCE the result is summed over
 * all ranks (reading R10: a SUM, not a mean). dw: DC_DW fp32. */
dc_status_t dc_conv_bwd_filter(dc_plan_t plan, const void *x_margined, const void *dy_margined,
                               float *dw, unsigned flags, void *stream);

/* Whole backward of the layer with the paper's overlap (PAPER.md:143, 177,
 * 204): dy halo exchange concurrent with backward-filter, then
 * backward-data, with the dW allreduce concurrent with backward-data.
 * Equivalent to dc_conv_bwd_filter + dc_conv_bwd_data with the same flags. */
dc_status_t dc_conv_bwd(dc_plan_t plan, const void *x_margined, void *dy_margined,
                        const void *w, void *dx, float *dw, unsigned flags, void *stream);

/* Spatially-aggregated batch-norm statistics (reading R11):
 * per channel, mean and biased variance of `t` over the local samples and
 * the whole spatial extent of the ranks that share this rank's samples
 * (equal i_N). t is a dense NHWC tensor (bf16, or fp32 for DC_FP32_3XTF32
 * plans) of the DC_Y layout of this plan
 * (channels = F, padded); mean_dev/var_dev are device fp64 arrays of F
 * entries. COLLECTIVE over the spatial group (each group of <= 8 ranks uses
 * its own one-shot NVLink mailbox of this plan; NCCL beyond).
 * flags: DC_BN_LOCAL gives the purely local variant ("purely
 * local batch normalization"; no communication). DC_BN_FROM_FWD states that
 * t is the y of this plan's most recent dc_conv_fwd, which ran with
 * DC_BN_STATS, and that t has not been written since: the per-CTA partials
 * that forward's epilogue accumulated are reduced instead of re-reading t
 * (same result up to fp64 summation order). The partials are used once;
 * without the flag, or when that forward could not accumulate them (another
 * forward of this plan ran since, or its launch shape has no fused
 * epilogue), t is read. Errors: DC_ERR_ARG (unknown flag), DC_ERR_COMM. */
#define DC_BN_LOCAL    0x1u
#define DC_BN_FROM_FWD 0x2u
dc_status_t dc_bn_spatial_stats(dc_plan_t plan, const void *t, double *mean_dev,
                                double *var_dev, unsigned flags, void *stream);

/* ---- the layers between the convolutions ---- */
#define DC_RELU 0x4u
/* Batch-norm apply on this rank's shard of a layer output y (DC_Y layout of
 * `plan`, bf16 or fp32 per the plan), with the group statistics mean / var
 * (device fp64 [F], from dc_bn_spatial_stats) and gamma / beta (device fp32
 * [F]): out = gamma (y - mean) / sqrt(var + eps) + beta [+ residual (DC_Y
 * layout)] [then ReLU with DC_RELU] (reading R27).
 * The result goes straight into the next layer's margined input when
 * dst_plan is given (dst = its DC_X buffer; its owned block must be this
 * plan's output block -- the same decomposition of the activation, else
 * DC_ERR_PARTITION -- fp32 plans store the [hi | lo] split), or to dst as a
 * dense tensor of the DC_Y layout. Elementwise, stream-ordered, not
 * collective. y and residual are read by bulk copies: 16-byte aligned device
 * pointers (torch allocations are), else DC_ERR_ARG. Errors: DC_ERR_ARG,
 * DC_ERR_PARTITION, DC_ERR_UNSUPPORTED (more than 3072 padded channels). */
dc_status_t dc_bn_apply(dc_plan_t plan, const void *y, const double *mean, const double *var, const float *gamma,
                        const float *beta, double eps, const void *residual, unsigned flags, dc_plan_t dst_plan,
                        void *dst, void *stream);
/* Backward of dc_bn_apply: dout = the gradient of its output (DC_Y layout of
 * `plan`, e.g. the next layer's dx), y / mean / var / gamma / beta / eps /
 * residual / flags as in the forward. With g = dout masked by the ReLU
 * (recomputed from y) and y_hat = (y - mean) / sqrt(var + eps), the sums
 * sum(g) and sum(g y_hat) are aggregated over the spatial group of the
 * forward statistics (COLLECTIVE over that group; DC_BN_LOCAL
 * for the purely local variant) and dy = gamma / sqrt(var + eps) (g - sum g
 * / M - y_hat sum(g y_hat) / M), M = the group's pixels, is written into
 * the owned block of dy_margined (this plan's DC_DY buffer, ready for the
 * dy halo exchange of the convolution's backward). dgamma = sum(g y_hat),
 * dbeta = sum g (device fp32 [F], may be NULL); dresidual (DC_Y layout, may
 * be NULL) receives g. dout, y and residual: 16-byte aligned device
 * pointers. Errors: DC_ERR_ARG, DC_ERR_COMM, DC_ERR_UNSUPPORTED (more than
 * 3072 padded channels). */
dc_status_t dc_bn_backward(dc_plan_t plan, const void *dout, const void *y, const double *mean, const double *var,
                           const float *gamma, const float *beta, double eps, const void *residual, unsigned flags,
                           float *dgamma, float *dbeta, void *dresidual, void *dy_margined, void *stream);

/* ---- redistribution between decompositions ----
 * Shuffle(D_i, D_j): when consecutive layers use different grids, each
 * activation (and, backward, each gradient) moves from the owned blocks of
 * one decomposition to those of the other; the element (n, c, h, w) goes from
 * its owner under D_i to its owner under D_j, every channel, nothing else.
 * The destination's margins are NOT filled (the next layer's halo exchange
 * does that). */
typedef struct dc_redist_s *dc_redist_t;
/* COLLECTIVE over the plans' communicator (virtual plans: host-only
 * geometry for dc_redist_bytes). Source: tensor tf (DC_Y / DC_DX: the dense
 * owned shard; DC_X / DC_DY: the owned interior of the margined buffer) of
 * plan `from`; destination: tensor tt of plan `to` (the owned interior of the
 * margined DC_X / DC_DY, or the dense DC_Y / DC_DX), whose dc_buffer_alloc
 * buffer must exist on every rank before this call (it is mapped into the
 * senders for the direct transport). The two tensors must have the same global N, H, W, channels
 * and pixel layout (fp32 plans: margined source only, DC_ERR_UNSUPPORTED
 * otherwise). Errors: DC_ERR_ARG, DC_ERR_SHAPE, DC_ERR_UNSUPPORTED. */
dc_status_t dc_redist_create(dc_plan_t from, dc_tensor_t tf, dc_plan_t to, dc_tensor_t tt, dc_redist_t *out);
/* Bytes this rank sends to / receives from each rank (arrays of world
 * entries; the block a rank keeps appears at its own index). */
dc_status_t dc_redist_bytes(dc_redist_t r, int64_t *send_bytes, int64_t *recv_bytes);
/* COLLECTIVE, stream-ordered. Moves src (the source shard, layout of tf)
 * into dst (the destination plan's dc_buffer_alloc buffer of tt). Default
 * transport: ONE kernel per rank stores every piece straight into its new
 * owner's buffer over NVLink peer memory, after that owner's ready flag, and
 * returns when every piece for this rank has arrived (device epochs, CUDA
 * graph replayable; <= 8 ranks). flags = DC_HALO_NCCL: pack, grouped
 * ncclSend / ncclRecv, unpack (real ranks; dst may then be any buffer of the
 * tt layout). src and dst may be reused / read after the call on `stream`.
 * Errors: DC_ERR_ARG, DC_ERR_UNSUPPORTED, DC_ERR_COMM, DC_ERR_CUDA. */
dc_status_t dc_redistribute(dc_redist_t r, const void *src, void *dst, unsigned flags, void *stream);
dc_status_t dc_redist_destroy(dc_redist_t r);

/* ---- channel / filter parallelism ----
 * A p_N x p_C grid of ranks (rank = i_N p_C + i_C): rank (i_N, i_C) owns the
 * samples block i_N and, of the channel dimensions, the input-channel block
 * i_C of x / dx / dW and the filter block i_C of y / dy ("if the input x is
 * partitioned on its C dimension, the output y is partitioned on its F
 * dimension"). Blocks are equal: C and F multiples of 16 p_C;
 * bf16 plans; the filter bank w is replicated (every rank holds all of it).
 *   forward:         y[F_r] = sum over the group's channel blocks of the
 *                    partial convolutions -- a reduce-scatter over F
 *                     fused into the conv GEMM: its epilogue
 *                    stores each fp32 partial tile into the owner's receive
 *                    slot over peer memory; the owner sums the p_C slots in
 *                    rank order and rounds to bf16 once;
 *   backward-data:   dx[C_r] likewise, a reduce-scatter over C;
 *   backward-filter: dy gathered over the group ("may require
 *                    data to be gathered"; one P2P all-to-all launch), then
 *                    dW[:, C_r] locally; DC_ALLREDUCE sums it over the p_N
 *                    sample groups (NCCL; real ranks).
 * All local tensors are dense NHWC without margins (dc_cplan_query). */
typedef struct dc_cplan_s *dc_cplan_t;
/* COLLECTIVE (comm of p_N p_C ranks, or NULL for 1 x 1). Errors: DC_ERR_ARG,
 * DC_ERR_SHAPE, DC_ERR_PARTITION, DC_ERR_UNSUPPORTED (fp32, C or F not a
 * multiple of 16 p_C, p_C > 8), DC_ERR_COMM. */
dc_status_t dc_cplan_create(int64_t N, int64_t C, int64_t H, int64_t W, int64_t F, int K, int stride, int pad,
                            int pn, int pc, dc_dtype_t dtype, dc_comm_t comm, dc_cplan_t *out);
/* Host-only geometry of rank `rank` (dc_cplan_query only). */
dc_status_t dc_cplan_create_virtual(int64_t N, int64_t C, int64_t H, int64_t W, int64_t F, int K, int stride,
                                    int pad, int pn, int pc, int rank, dc_cplan_t *out);
/* Local shard of t: X / DX [n][H][W][C_r], Y / DY [n][Ho][Wo][F_r], W the
 * whole [F][K][K][C] bf16 bank, DW [F][K][K][C_r] fp32; *c0 (may be NULL) =
 * the first global channel (X, DX, DW: of C; Y, DY: of F; W: 0). */
dc_status_t dc_cplan_query(dc_cplan_t plan, dc_tensor_t t, dc_shard_desc_t *desc, int64_t *c0);
/* COLLECTIVE over the channel group, stream-ordered; flags 0. */
dc_status_t dc_cconv_fwd(dc_cplan_t plan, const void *x, const void *w, void *y, unsigned flags, void *stream);
dc_status_t dc_cconv_bwd_data(dc_cplan_t plan, const void *dy, const void *w, void *dx, unsigned flags,
                              void *stream);
/* flags: 0 or DC_ALLREDUCE. */
dc_status_t dc_cconv_bwd_filter(dc_cplan_t plan, const void *x, const void *dy, float *dw, unsigned flags,
                                void *stream);
dc_status_t dc_cplan_destroy(dc_cplan_t plan);

/* ---- max pooling on the decomposition ----
 * "Pooling layers are parallelized similarly" to convolution,
 * with "halo exchanges before ... pooling": window K (odd, as
 * for the convolutions), stride,
 * pad (out-of-range positions are not part of a window), the same blocked
 * sample x spatial grid as a convolution. The gradient of a window goes to
 * its FIRST maximum in (a, b) order. bf16 plans.
 * The pooling owns two plans of its grid: `in_plan` holds the input x as a
 * margined DC_X buffer with a halo of K - 1 on every side (allocate it with
 * dc_buffer_alloc(in_plan, DC_X); dc_bn_apply may write into it with
 * dst_plan = in_plan), and `out_plan` describes y (DC_Y, dense), dy (DC_DY,
 * margined: dc_buffer_alloc(out_plan, DC_DY)) and dx (DC_DX, dense). The
 * backward recomputes each window's first maximum from the wide x, so no
 * argmax tensor is stored or exchanged. */
typedef struct dc_pool_s *dc_pool_t;
/* COLLECTIVE. decomp entries must all be > 0. Errors: DC_ERR_ARG,
 * DC_ERR_SHAPE, DC_ERR_PARTITION (a window of an owned output reaches past
 * the neighbouring input blocks), DC_ERR_UNSUPPORTED (fp32, 2K - 1 > 15). */
dc_status_t dc_pool_create(int64_t N, int64_t C, int64_t H, int64_t W, int K, int stride, int pad, dc_decomp_t decomp,
                           dc_dtype_t dtype, dc_comm_t comm, dc_pool_t *out);
dc_status_t dc_pool_plans(dc_pool_t pool, dc_plan_t *in_plan, dc_plan_t *out_plan);
/* y = maxpool(x) on the owned outputs; flags DC_EXCHANGE: exchange x's halo
 * first (x must then be in_plan's dc_buffer_alloc buffer; | DC_HALO_NCCL). */
dc_status_t dc_pool_fwd(dc_pool_t pool, void *x, void *y, unsigned flags, void *stream);
/* dx on the owned inputs from dy (out_plan's margined dy; DC_EXCHANGE
 * exchanges its halo first) and x (with its halo, as the forward left it). */
dc_status_t dc_pool_bwd(dc_pool_t pool, const void *x, void *dy, void *dx, unsigned flags, void *stream);
dc_status_t dc_pool_destroy(dc_pool_t pool);

/* Number of kernels this library launched on this thread so far (for the
 * bench's gpu_launches claim). */
uint64_t dc_kernel_launches(void);

/* Thread-local message of the last failing call (valid until the next call
 * on the same thread). */
const char *dc_last_error(void);

/* ---- performance model, host only ---- */
/* alpha [s], beta [s/byte] of the linear point-to-point model. */
dc_status_t dc_model_set_comm(double alpha, double beta);
/* Overlap accounting of the model ("adjusting for overlap if
 * necessary"): 1 (default) = reading R16, FP = max(C, halo_x), BP = max(Cw,
 * halo_dy) + max(Cx, BPa); 0 = plain sums (every exchange exposed), for an
 * implementation whose measured exchanges are not hidden. */
dc_status_t dc_model_set_overlap(int overlap);
/* Extra latency [s] added to every east/west and corner halo message of the
 * model (default 0 = the paper's SR for all messages): in
 * NHWC those slabs are H_l strided runs rather than one contiguous block, and
 * their boundary tiles are column strips (measured). */
dc_status_t dc_model_set_strided_latency(double alpha_w);
/* Load an empirical cost table (CSV "op,n,c,h,w,f,k,s,pad,seconds",
 * op in {fp,bpx,bpw}). Entries missing from the table
 * fall back to a roofline estimate. */
dc_status_t dc_model_load_table(const char *csv_path);
/* Predicted seconds of fwd+bwd of the layer on grid d (PAPER.md:190-206,
 * overlap per reading R16); returns DC_ERR_PARTITION if d is invalid. */
dc_status_t dc_model_layer_cost(int64_t N, int64_t C, int64_t H, int64_t W, int64_t F, int K,
                                int stride, int pad, dc_decomp_t d, int include_allreduce,
                                double *seconds);
/* Argmin over all valid grids of `world` ranks (tie-break reading R17). */
dc_status_t dc_model_choose(int64_t N, int64_t C, int64_t H, int64_t W, int64_t F, int K,
                            int stride, int pad, int world, dc_decomp_t *best, double *seconds);
/* The same argmin over the grids whose entries equal fix's non-zero entries
 * (e.g. fix = {1,0,0}: the best pure spatial grid, BASELINE configs[3]);
 * what dc_plan_create does with a partly-zero decomp. DC_ERR_PARTITION if no
 * valid grid matches. */
dc_status_t dc_model_choose_fixed(int64_t N, int64_t C, int64_t H, int64_t W, int64_t F, int K,
                                  int stride, int pad, int world, dc_decomp_t fix, dc_decomp_t *best,
                                  double *seconds);

/* ---- parallel execution strategies (NEXT-3) ---- */
/* Shuffle(D_i, D_j): seconds to move an N x Ch x H x W activation (2-byte
 * words) from grid `from`'s blocked distribution to grid `to`'s with a
 * pairwise-exchange all-to-all -- the max over ranks of the sum over peers of
 * SR(words sent); 0 when the grids agree. */
dc_status_t dc_model_shuffle_cost(int64_t N, int64_t Ch, int64_t H, int64_t W, dc_decomp_t from, dc_decomp_t to,
                                  double *seconds);
/* One layer of a network for dc_model_strategy: its conv shape and the layers
 * whose outputs it reads (-1: none / the network input; a residual join has
 * two parents; shapes must chain: parent F, Ho, Wo = this C, H, W). */
typedef struct {
    int64_t N, C, H, W, F;
    int32_t K, stride, pad;
    int32_t parent, parent2;
} dc_layer_t;
/* A parallel execution strategy: one grid per layer minimising the sum of the
 * layers' Cost_D(l) (dc_model_layer_cost) and the shuffles of every edge,
 * forward and backward (reading R28). A line network is solved
 * exactly by the shortest path over per-layer candidates;
 * with branches, the longest remaining path is solved first and fixed, and
 * so on. fix_pn > 0 restricts the candidates to p_N = fix_pn
 * (1: pure spatial). grids: n entries out; total_seconds (may be NULL): the
 * strategy's model time. Errors: DC_ERR_ARG, DC_ERR_SHAPE, DC_ERR_PARTITION. */
dc_status_t dc_model_strategy(const dc_layer_t *layers, int n, int world, int fix_pn, dc_decomp_t *grids,
                              double *total_seconds);

#ifdef __cplusplus
}
#endif
#endif /* DCONV_H */
