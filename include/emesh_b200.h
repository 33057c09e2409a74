/*
 * emesh_b200 — B200-native (sm_100a) outer-synchronisation hot path of the
 * INTELLECT-1 / PRIME DiLoCo stack, behind a plain C ABI.
 *
 * Drop-in boundary for the reference's C++ API in proj/include/emesh
 * (header-only C++20 library). Each entry point names the reference
 * interface it replaces. No torch types; plain pointers, sizes, CUDA
 * streams. Device pointers unless a name says _host. fp32 arenas the
 * quantizer reads (quantize input, ring input, theta_g / theta_l) must be
 * 32-byte aligned and code arenas 8-byte aligned (256-bit loads; cudaMalloc
 * gives 256); other fp32 arenas 16-byte aligned.
 *
 * Error convention (maps 1:1 onto the reference's exception hierarchy,
 * proj/include/emesh/errors.hpp:10-73): functions return EMESH_OK or an
 * EMESH_E* code; emesh_last_error() gives the message (thread-local).
 */
#ifndef EMESH_B200_H
#define EMESH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* emesh_stream_t; /* == cudaStream_t */

enum {
    EMESH_OK = 0,
    EMESH_ESHAPE = 1,   /* emesh::ShapeError   (size mismatch / empty chunk) */
    EMESH_ENUMERIC = 2, /* emesh::NumericError (non-finite input, quant.hpp:29-31) */
    EMESH_EDECODE = 3,  /* emesh::DecodeError  (malformed wire buffer, quant.hpp:117-131) */
    EMESH_ECUDA = 4,    /* CUDA runtime failure */
    EMESH_ENCCL = 5,    /* NCCL failure (the transport; emesh::LinkError analogue) */
    EMESH_ERING = 6,    /* emesh::RingFailureError (collective aborted) */
    EMESH_ECONFIG = 7,  /* emesh::ConfigError (invalid plan/options) */
    EMESH_EIO = 8,      /* emesh::Error (checkpoint file I/O, integrity hash mismatch) */
    EMESH_ESTALE = 9,   /* emesh::StalePlanError (a ring peer runs a newer plan epoch, allreduce.hpp:272) */
    EMESH_EPROTO = 10   /* emesh::Error "ring protocol violation" (unexpected chunk header, allreduce.hpp:280) */
};

#define EMESH_BUCKETS 256

const char* emesh_last_error(void);
int emesh_abi_version(void);

/* ---------------- codec: proj/include/emesh/quant.hpp ------------------ */

/* quant.hpp:28 `QuantChunk quantize(std::span<const float>)`: one segment
 * of n values -> n u8 codes + 256 f32 codebook. Synchronous on `stream`
 * (the reference throws synchronously): returns EMESH_ESHAPE for n == 0 and
 * EMESH_ENUMERIC for non-finite input. stats (optional, device, 4 doubles):
 * {mu, sigma, lo, width}. */
int emesh_quantize(const float* x, uint64_t n, uint8_t* codes, float* codebook, double* stats,
                   emesh_stream_t stream);

/* Batched form over a segment table (allreduce.hpp:326-336 sub-slices):
 * segment i is x[seg_lo[i] .. seg_lo[i]+seg_len[i]) with its codebook at
 * codebooks[i*256]. seg_lo/seg_len are HOST arrays. codes are written at the
 * same element offsets as x. Asynchronous; non-finite input is reported by
 * emesh_codec_check(). */
int emesh_quantize_segments(const float* x, const uint64_t* seg_lo, const uint64_t* seg_len,
                            uint32_t nseg, uint8_t* codes, float* codebooks, double* stats,
                            emesh_stream_t stream);
/* Synchronizes `stream`; EMESH_ENUMERIC if any quantize since the last check
 * saw a non-finite value. */
int emesh_codec_check(emesh_stream_t stream);

/* quant.hpp:89 `dequantize_into`: out[i] = codebook[codes[i]]. */
int emesh_dequantize(const uint8_t* codes, const float* codebook, uint64_t n, float* out,
                     emesh_stream_t stream);
int emesh_dequantize_segments(const uint8_t* codes, const float* codebooks, const uint64_t* seg_lo,
                              const uint64_t* seg_len, uint32_t nseg, float* out,
                              emesh_stream_t stream);

/* quant.hpp:102-131 wire layout (u32 LE count, 256 f32 LE, count u8), host
 * buffers: encode writes 1028+n bytes; decode validates like the reference
 * (EMESH_EDECODE on truncation, non-finite codebook, count mismatch). */
uint64_t emesh_encode_quant_chunk(const uint8_t* codes_host, const float* codebook_host, uint32_t n,
                                  uint8_t* out_host);
int emesh_decode_quant_chunk(const uint8_t* buf_host, uint64_t len, uint8_t* codes_host,
                             float* codebook_host, uint32_t* count);

/* ---------------- optimizer: proj/include/emesh/optim.hpp --------------- */

/* optim.hpp:99 `compute_pseudo_gradient`: delta = theta_prev - theta_local
 * over the flat canonical arena (tensor.hpp:87-93). */
int emesh_pseudo_gradient(const float* theta_prev, const float* theta_local, float* delta, uint64_t n,
                          emesh_stream_t stream);

/* optim.hpp:63-94 `adamw_step` on a flat arena (the inner step that produces
 * theta_l): `step` = AdamWState.step AFTER the increment (>= 1); bias
 * corrections use std::pow in double exactly as the reference. A non-finite
 * gradient sets bit 0 of *err_flag (device word, optional) and leaves that
 * element untouched; the caller raises NumericError. */
int emesh_adamw_step(float* params, const float* grads, float* m, float* v, uint64_t n, uint64_t step,
                     float inner_lr, float lr_scale, float beta1, float beta2, float eps, float weight_decay,
                     uint32_t* err_flag, emesh_stream_t stream);

/* optim.hpp:116 `nesterov_outer_step`: b = mu*b + d; theta -= lr*(d + mu*b). */
int emesh_nesterov_outer_step(float* theta, const float* avg_delta, float* momentum_buf, uint64_t n,
                              float outer_lr, float outer_momentum, emesh_stream_t stream);

/* ---------------- ring engine: proj/include/emesh/allreduce.hpp --------- */

typedef struct emesh_engine emesh_engine;

typedef struct {
    uint64_t n;                 /* params per worker (flat arena length) */
    uint32_t k;                 /* ring size = DiLoCo workers (RingPlan.order.size()) */
    uint32_t rank;              /* RingPlan.self_index (NCCL mode) */
    uint32_t pipeline_subchunks;/* ReduceOptions.pipeline_subchunks (S), default 4 */
    uint32_t virtual_workers;   /* 0/1: one worker per process over NCCL;
                                   == k: all k workers on this GPU (zero-copy ring) */
    uint64_t window_elems;      /* pipelining window (0 = auto) */
    const uint8_t* nccl_id;     /* 128-byte ncclUniqueId (NCCL mode, k > 1) */
    int device;                 /* CUDA device ordinal, -1 = current */
    uint32_t transport;         /* EMESH_TRANSPORT_*: how hop payloads move between ranks */
    uint32_t reduce_fp32;       /* ReduceJob.mode (allreduce.hpp:49-53, :120-164): 0 = ReduceMode::int8
                                   (uint8 codes + codebooks), 1 = ReduceMode::fp32 (raw fp32 partial sums).
                                   One engine serves one mode; make one per mode in use. */
    const uint64_t* tensor_numel; /* optional (ntensors > 0): the flat arena is this list of tensors
                                   (canonical order, sum = n) and each tensor is its own ReduceJob:
                                   k chunks x min(S, len) segments per tensor, all tensors' chunk c
                                   reduced together ("bucketing") */
    uint32_t ntensors;
    double step_timeout_s;      /* ReduceOptions.step_timeout (allreduce.hpp:59): a wait on a peer that
                                   exceeds it aborts the round and emesh_engine_check returns EMESH_ERING
                                   (RingFailureError) — peer transport: the kernels' spin budget; NCCL
                                   transport: the non-blocking communicator's enqueue / completion polls,
                                   after which it is aborted. 0 = 30 s. */
    uint32_t plan_epoch;        /* RingPlan.epoch (allreduce.hpp:25-45): carried in every payload's ChunkMsg
                                   header and compared at engine setup; a peer with a newer epoch ->
                                   EMESH_ESTALE (StalePlanError) */
} emesh_engine_config;

/* Transports of the one-process-per-GPU ring (k > 1, not virtual):
 *   AUTO: P2P when every rank's GPU is reachable through CUDA IPC peer memory
 *         (one NVLink / NVSwitch node), else NCCL;
 *   NCCL: ncclSend / ncclRecv of each window's codes + codebooks per hop;
 *   P2P:  the quantizer writes each hop's codes + codebooks straight into the
 *         successor's arena (the owner's final payload into every rank's)
 *         and raises a per-segment arrival flag there; the next hop's
 *         quantizer and the Nesterov apply wait on those flags segment by
 *         segment (NCCL only bootstraps the IPC handles). */
enum { EMESH_TRANSPORT_AUTO = 0, EMESH_TRANSPORT_NCCL = 1, EMESH_TRANSPORT_P2P = 2 };

/* Transport the engine resolved to (EMESH_TRANSPORT_NCCL / _P2P; 0 for the
 * virtual ring and k == 1). */
int emesh_engine_transport(const emesh_engine* e);

/* Host-only plan queries (no GPU needed). Segment table of an (n, k, S)
 * ring, chunk-major (allreduce.hpp:107-118, :326-336); returns the count. */
uint64_t emesh_plan_segments(uint64_t n, uint32_t k, uint32_t S, uint64_t* seg_lo, uint64_t* seg_len);
/* Same for a multi-tensor engine (emesh_engine_config.tensor_numel): chunk-major, tensors in order. */
uint64_t emesh_plan_tensor_segments(const uint64_t* tensor_numel, uint32_t ntensors, uint32_t k, uint32_t S,
                                    uint64_t* seg_lo, uint64_t* seg_len);

/* The NCCL ring engine's program for one ring position, in issue order.
 * kinds: OWN = quantize own chunk's hop-0 payload window; XFER = send
 * window of send_chunk to rank+1 and receive the window of recv_chunk from
 * rank-1; QUANT = fused dequant+add+requant of the received window
 * (final_hop: owner mean /k, allreduce.hpp:435-443); APPLY = decode a final
 * window (dequant + Nesterov). Windows are ranges of segment slots. */
enum { EMESH_OP_OWN = 0, EMESH_OP_XFER = 1, EMESH_OP_QUANT = 2, EMESH_OP_APPLY = 3 };
typedef struct {
    int32_t kind, phase, hop, window;  /* phase 0 reduce-scatter, 1 all-gather */
    int32_t send_chunk, recv_chunk;     /* -1 when unused */
    uint32_t send_seg0, send_nseg, recv_seg0, recv_nseg;
    int32_t final_hop, pad;
} emesh_ring_op;
uint64_t emesh_ring_schedule(uint64_t n, uint32_t k, uint32_t S, uint64_t window_elems, uint32_t rank,
                             emesh_ring_op* ops, uint64_t max_ops);

/* NCCL unique id for emesh_engine_config.nccl_id (rank 0 creates, broadcast). */
int emesh_nccl_unique_id(uint8_t out[128]);

/* RingPlan + ReduceOptions (allreduce.hpp:25-62): builds the segment table,
 * the pipelining windows, all device scratch (no allocation afterwards) and
 * the NCCL communicator. */
int emesh_engine_create(const emesh_engine_config* cfg, emesh_engine** out);
int emesh_engine_destroy(emesh_engine* e);

/* Segment table (allreduce.hpp:107-118,326-336), chunk-major; returns the
 * count, fills lo/len when non-NULL (host arrays). */
uint64_t emesh_engine_segments(const emesh_engine* e, uint64_t* seg_lo, uint64_t* seg_len);

/* allreduce.hpp:314 `ring_allreduce` (ReduceMode::int8): output = the
 * elementwise mean of the workers' inputs as every rank decodes it. Inputs
 * are preserved (ReduceJob contract, allreduce.hpp:47-48). Arrays have one
 * entry per local worker (1 in NCCL mode, k in virtual mode). */
int emesh_engine_ring_allreduce(emesh_engine* e, const float* const* input, float* const* output,
                                emesh_stream_t stream);

/* One DiLoCo outer sync (trainer.hpp:355-382): delta = theta_g - theta_l
 * (never materialized) -> int8 ring all-reduce -> Nesterov fused with the
 * final dequantize; theta_g and momentum_buf updated in place; with
 * write_local, theta_l <- theta_g (trainer.hpp:382). */
int emesh_engine_outer_sync(emesh_engine* e, float* const* theta_g, float* const* theta_l,
                            float* const* momentum_buf, float outer_lr, float outer_momentum,
                            int write_local, emesh_stream_t stream);

/* Same round with HOST buffers (what the reference's Trainer holds):
 * H2D of theta_g/theta_l/momentum_buf, the round, D2H of the updated
 * theta_g/momentum_buf (+theta_l with write_local). Synchronous. Pinned
 * host memory gives full PCIe bandwidth. */
int emesh_engine_outer_sync_host(emesh_engine* e, float* const* theta_g, float* const* theta_l,
                                 float* const* momentum_buf, float outer_lr, float outer_momentum,
                                 int write_local);

/* Synchronizes the engine; EMESH_ENUMERIC if a quantize saw non-finite data
 * since the last check (the reference's NumericError, quant.hpp:31).
 * Ring failures (peer transport; allreduce.hpp:247-305, :341-359, :466-472):
 * EMESH_ERING (RingFailureError: a peer stalled past step_timeout or a
 * poisoned flag swept the failure around the ring), EMESH_ESTALE
 * (StalePlanError), EMESH_EPROTO (protocol violation). A failed round
 * commits NOTHING on any rank (theta_g / momentum / theta_l untouched), so
 * allreduce_with_retry can restart from the same state; the engine is then
 * unusable (rebuild it over the survivors). */
int emesh_engine_check(emesh_engine* e);

/* The rank the last failed round names as the culprit (the predecessor whose
 * reduce-scatter payload or the owner whose final payload never arrived, or
 * the one a poisoned flag names; a waiter whose predecessor is itself
 * waiting in the round first gives it one more step_timeout for its verdict);
 * -1 when unknown — always past k = 2 on the NCCL transport, which has no
 * abort frames. RingFailureError.failed_node. */
int emesh_engine_failed_rank(const emesh_engine* e);

/* ReduceJob.id of the engine's next round (ChunkMsg job id; default: the
 * engine's round counter). */
int emesh_engine_set_job(emesh_engine* e, uint64_t job_id);

/* Device views of a local worker's final payload arenas after a round:
 * codes (n bytes, arena-indexed) and codebooks (nseg x 256). In NCCL mode
 * every chunk's final payload is present (the all-gather delivered it); in
 * virtual mode chunk c's lives in worker (c-1)%k's arena. */
int emesh_engine_payload(emesh_engine* e, uint32_t worker, const uint8_t** codes, const float** codebooks,
                         const double** seg_stats, uint64_t* stats_stride_bytes);

/* Host copies of the same: codes (n bytes), codebooks (nseg*256 f32),
 * stats (nseg*4 f64: mu, sigma, lo, width). Synchronizes the engine. */
int emesh_engine_payload_host(emesh_engine* e, uint32_t worker, uint8_t* codes_host, float* codebooks_host,
                              double* stats_host);

/* Number of kernels this engine launched since creation (for the bench's
 * gpu_launches claim). */
uint64_t emesh_engine_launches(const emesh_engine* e);

/* Per-kernel profiling with CUDA events on the launching stream. enable
 * resets the record. kind: 0, 1 reserved, 2 hop-0 quantize, 3 RS hop
 * quantize, 4 owner-final quantize, 5 plain quantize, 6 dequant + Nesterov,
 * 7 dequantize, 8 k==1 fused PG+Nesterov, 9 fp32-mode hop, 10 fp32-mode
 * decode (+ Nesterov). Reads launches, total device ms and total
 * ALGORITHMIC bytes of that kind. */
int emesh_engine_profile(emesh_engine* e, int enable);
int emesh_engine_profile_read(emesh_engine* e, uint32_t kind, uint64_t* launches, double* ms, double* alg_bytes);

/* NCCL-mode op timeline of the calls made since emesh_engine_profile(e, 1):
 * rows of 6 doubles {op kind, phase, hop, window, start ms, end ms} (times on
 * the op's stream, relative to the first op's start). Returns the row count
 * (copies at most max_rows). Synchronizes the engine. */
uint64_t emesh_engine_timeline(emesh_engine* e, double* rows, uint64_t max_rows);

/* ---------------- checkpoints: tensor.hpp:111-161, checkpoint.hpp:19-68,190-224 ----
 * A Checkpoint whose five parameter sets stay in device arenas (flat fp32,
 * canonical tensor order, `numel` = sum of the tensors' element counts each).
 * The layout (names, ranks, extents) is the model's; the bytes are exactly
 * encode_checkpoint's (checkpoint.hpp:32-47). Names are NUL-terminated UTF-8. */
typedef struct emesh_checkpoint {
    uint64_t outer_step;
    uint32_t ntensors;
    const char* const* names;   /* ntensors */
    const uint32_t* ranks;      /* ntensors */
    const uint32_t* extents;    /* sum(ranks), tensor after tensor */
    float* params;              /* Checkpoint::params (theta after the outer step) */
    float* retained;            /* Checkpoint::retained (theta_g for the next pseudo-gradient) */
    float* adam_m;              /* Checkpoint::inner.m */
    float* adam_v;              /* Checkpoint::inner.v */
    float* nesterov_buf;        /* Checkpoint::outer.buffer */
    uint64_t adam_step;         /* Checkpoint::inner.step */
    uint64_t rng_seed;
    uint64_t data_counter;
    uint32_t shard;
    uint8_t config_hash[32];
} emesh_checkpoint;

/* Size of encode_checkpoint(ck) in bytes. */
int emesh_checkpoint_encoded_size(const emesh_checkpoint* ck, uint64_t* bytes);
/* checkpoint.hpp:32-47 into a host buffer (page-locked: DMA in place; else
 * staged through pinned blocks). EMESH_ESHAPE if cap is short (*written = need). */
int emesh_checkpoint_encode(const emesh_checkpoint* ck, uint8_t* out_host, uint64_t cap, uint64_t* written,
                            emesh_stream_t stream);
/* checkpoint.hpp:49-66 into the view's arenas: the same DecodeError /
 * ShapeError cases as the reference (first one in stream order), plus
 * EMESH_EDECODE when the bytes' layout differs from the view's. Scalars are
 * written back into *ck. Structural errors leave the arenas untouched; a
 * non-finite value is detected on the device after the upload. */
int emesh_checkpoint_decode(const uint8_t* buf_host, uint64_t len, emesh_checkpoint* ck, emesh_stream_t stream);
/* Layout discovery (the params set): counts, then names (NUL-separated),
 * ranks and extents. */
int emesh_checkpoint_probe(const uint8_t* buf_host, uint64_t len, uint32_t* ntensors, uint64_t* numel,
                           uint64_t* name_bytes, uint32_t* rank_sum);
int emesh_checkpoint_layout(const uint8_t* buf_host, uint64_t len, char* names, uint64_t names_cap,
                            uint32_t* ranks, uint32_t* extents, uint32_t extents_cap);
/* checkpoint.hpp:190-224 file framing: u64 LE length, sha256(payload),
 * payload. read: EMESH_EIO on open failure / hash mismatch, EMESH_EDECODE on
 * truncation, then emesh_checkpoint_decode. */
int emesh_checkpoint_write_file(const char* path, const emesh_checkpoint* ck, emesh_stream_t stream);
int emesh_checkpoint_read_file(const char* path, emesh_checkpoint* ck, emesh_stream_t stream);
/* sha256.hpp: one-shot SHA-256 (host). */
int emesh_sha256(const void* data, uint64_t n, uint8_t out[32]);

#ifdef __cplusplus
}
#endif
#endif /* EMESH_B200_H */
